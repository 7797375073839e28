/* demc_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE (see demc_oracle.h).
 *
 * Plain-C restatement of the reference compile pipeline. Every function cites
 * the reference file:line it follows (paths relative to
 * /root/reference/proj/core/src/). Not reentrant (single-threaded checker).
 */
#define _GNU_SOURCE
#include "demc_oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define NO_SUCC 0xFFFFFFFFu /* kNoSuccessor, stepg.hpp:52 */

static char g_err[256];
const char *oracle_last_error(void) { return g_err; }

static int fail(int code, const char *msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

/* ---- util ------------------------------------------------------------- */

/* dem.cpp:27-37: FNV-1 64 over words, LSB-first bytes, multiply then XOR. */
uint64_t oracle_fnv1_64(const uint64_t *words, size_t n) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < n; i++)
        for (int b = 0; b < 8; b++) {
            h *= 0x100000001b3ull;
            h ^= (words[i] >> (8 * b)) & 0xff;
        }
    return h;
}

/* dem.hpp:28-30 (compiled with -ffp-contract=off: no FMA). */
double oracle_merge_prob(double a, double b) { return a * (1 - b) + b * (1 - a); }

/* ---- sources: stepg.cpp:49-121 ---------------------------------------- */

enum { P_X = 0, P_Y = 1, P_Z = 2 };
enum { G_H = 0, G_CX = 1, G_R = 2, G_M = 3, G_MR = 4 };
enum { N_XERR = 0, N_ZERR = 1, N_DEP1 = 2, N_DEP2 = 3 };

typedef struct {
    double prob;
    int32_t boundary; /* -1 for measurement flips */
    int32_t measurement;
    uint32_t nterms;
    uint32_t q[2];
    uint8_t p[2];
} spec_t; /* SourceSpec, stepg.hpp:45-50 */

/* kPairTable, stepg.cpp:49-58: the 15 two-qubit Paulis with the level that
 * first retains them. 'I' = identity component. */
static const char kPairs[15][3] = {
    {'I', 'X', 0}, {'I', 'Y', 1}, {'I', 'Z', 0}, {'X', 'I', 0}, {'X', 'X', 0},
    {'X', 'Y', 2}, {'X', 'Z', 1}, {'Y', 'I', 1}, {'Y', 'X', 2}, {'Y', 'Y', 2},
    {'Y', 'Z', 2}, {'Z', 'I', 0}, {'Z', 'X', 1}, {'Z', 'Y', 2}, {'Z', 'Z', 0},
};

static uint8_t pauli_of(char c) { return c == 'X' ? P_X : c == 'Y' ? P_Y : P_Z; }

typedef struct {
    spec_t *v;
    size_t n, cap;
} specs_t;

static int push_spec(specs_t *s, spec_t x) {
    if (s->n == s->cap) {
        size_t nc = s->cap ? 2 * s->cap : 1024;
        spec_t *nv = realloc(s->v, nc * sizeof *nv);
        if (!nv) return 0;
        s->v = nv;
        s->cap = nc;
    }
    s->v[s->n++] = x;
    return 1;
}

/* decompose_noise (stepg.cpp:66-103) + enumerate_sources (stepg.cpp:105-121):
 * per layer, noise ops first, then M/MR flips with flip_prob > 0. */
static int enumerate_sources(const oracle_circuit *c, int level, specs_t *out) {
    for (uint32_t i = 0; i < c->num_layers; i++) {
        for (uint32_t o = c->noise_offsets[i]; o < c->noise_offsets[i + 1]; o++) {
            spec_t s;
            memset(&s, 0, sizeof s);
            s.boundary = (int32_t)i;
            s.measurement = -1;
            uint32_t q0 = c->noise_q0[o], q1 = c->noise_q1[o];
            double p = c->noise_prob[o];
            switch (c->noise_kind[o]) {
                case N_XERR:
                case N_ZERR:
                    s.prob = p;
                    s.nterms = 1;
                    s.q[0] = q0;
                    s.p[0] = c->noise_kind[o] == N_XERR ? P_X : P_Z;
                    if (!push_spec(out, s)) return 0;
                    break;
                case N_DEP1: {
                    s.prob = p / 3;
                    s.nterms = 1;
                    s.q[0] = q0;
                    s.p[0] = P_X;
                    if (!push_spec(out, s)) return 0;
                    if (level != 0) {
                        s.p[0] = P_Y;
                        if (!push_spec(out, s)) return 0;
                    }
                    s.p[0] = P_Z;
                    if (!push_spec(out, s)) return 0;
                    break;
                }
                case N_DEP2: {
                    s.prob = p / 15;
                    for (int t = 0; t < 15; t++) {
                        if (kPairs[t][2] > level) continue;
                        s.nterms = 0;
                        if (kPairs[t][0] != 'I') {
                            s.q[s.nterms] = q0;
                            s.p[s.nterms++] = pauli_of(kPairs[t][0]);
                        }
                        if (kPairs[t][1] != 'I') {
                            s.q[s.nterms] = q1;
                            s.p[s.nterms++] = pauli_of(kPairs[t][1]);
                        }
                        if (!push_spec(out, s)) return 0;
                    }
                    break;
                }
            }
        }
        for (uint32_t g = c->gate_offsets[i]; g < c->gate_offsets[i + 1]; g++) {
            uint8_t k = c->gate_kind[g];
            if ((k == G_M || k == G_MR) && c->gate_flip[g] > 0) {
                spec_t s;
                memset(&s, 0, sizeof s);
                s.prob = c->gate_flip[g];
                s.boundary = -1;
                s.measurement = c->gate_meas[g];
                if (!push_spec(out, s)) return 0;
            }
        }
    }
    return 1;
}

/* ---- lowering: stepg.cpp:165-315 -------------------------------------- */

typedef struct {
    uint32_t node0, node1;
    double prob;
} source_t; /* ErrorSource, stepg.hpp:55-60 */

typedef struct {
    uint32_t n, l, k, M, D, O;
    int level;
    uint64_t *succ; /* l*k packed (lo = first, hi = second), stepg.hpp:85-91 */
    source_t *src;
    size_t S;
} stepg_t;

/* SlotLayout, stepg.hpp:96-112 */
#define X_SLOT(q) (2 * (q))
#define Z_SLOT(q) (2 * (q) + 1)
#define Y_SLOT(q) (2 * n + (q))
#define XZ_SLOT(j) (3 * n + 2 * (j))
#define ZX_SLOT(j) (3 * n + 2 * (j) + 1)
#define XY_SLOT(j) (4 * n + 5 * (j))
#define YX_SLOT(j) (4 * n + 5 * (j) + 1)
#define YY_SLOT(j) (4 * n + 5 * (j) + 2)
#define YZ_SLOT(j) (4 * n + 5 * (j) + 3)
#define ZY_SLOT(j) (4 * n + 5 * (j) + 4)

static uint64_t pack2(uint32_t a, uint32_t b) { return (uint64_t)b << 32 | a; }

static int lower(const oracle_circuit *c, int level, stepg_t *g) {
    const uint32_t n = c->num_qubits, l = c->num_layers;
    const uint32_t alpha = level == 0 ? 2 : level == 1 ? 4 : 7; /* stepg.cpp:23-33 */
    const uint32_t k = alpha * n;
    uint64_t rows = (uint64_t)l * k + c->num_measurements;
    if (rows >= NO_SUCC) return fail(1, "circuit exceeds 32-bit node index space");
    memset(g, 0, sizeof *g);
    g->n = n;
    g->l = l;
    g->k = k;
    g->M = c->num_measurements;
    g->D = c->num_detectors;
    g->O = c->num_observables;
    g->level = level;
    g->succ = malloc(((size_t)l * k + 1) * sizeof(uint64_t));
    if (!g->succ) return fail(4, "out of memory");
    for (size_t u = 0; u < (size_t)l * k; u++) g->succ[u] = pack2(NO_SUCC, NO_SUCC);
#define NODE(b, s) ((uint32_t)((b) * k + (s)))
#define LEAF(m) ((uint32_t)(l * k + (m)))

    /* index_layer (stepg.cpp:139-161), flattened to per-qubit arrays:
     * kind (-1 idle), partner, control flag, meas index; CX (c,t) -> j via the
     * control qubit (validated circuits touch each qubit at most once). */
    int8_t *kind = malloc((size_t)l * n + 1);
    uint32_t *partner = malloc(((size_t)l * n + 1) * sizeof(uint32_t));
    uint8_t *ctrl = malloc((size_t)l * n + 1);
    int32_t *meas = malloc(((size_t)l * n + 1) * sizeof(int32_t));
    int32_t *cxj = malloc(((size_t)l * n + 1) * sizeof(int32_t)); /* j of CX controlled by q */
    if (!kind || !partner || !ctrl || !meas || !cxj) return fail(4, "out of memory");
    memset(kind, -1, (size_t)l * n);
    for (size_t t = 0; t < (size_t)l * n; t++) cxj[t] = -1;
    for (uint32_t i = 0; i < l; i++) {
        uint32_t j = 0;
        for (uint32_t gi = c->gate_offsets[i]; gi < c->gate_offsets[i + 1]; gi++) {
            uint32_t q0 = c->gate_q0[gi], q1 = c->gate_q1[gi];
            size_t a = (size_t)i * n + q0;
            kind[a] = (int8_t)c->gate_kind[gi];
            if (c->gate_kind[gi] == G_CX) {
                size_t b = (size_t)i * n + q1;
                partner[a] = q1;
                ctrl[a] = 1;
                cxj[a] = (int32_t)(j++);
                kind[b] = G_CX;
                partner[b] = q0;
                ctrl[b] = 0;
            } else if (c->gate_kind[gi] == G_M || c->gate_kind[gi] == G_MR) {
                meas[a] = c->gate_meas[gi];
            }
        }
    }

    for (uint32_t i = 0; i < l; i++) {
        /* Base X/Z slots through layer i+1 (stepg.cpp:196-234). */
        if (i + 1 < l) {
            for (uint32_t q = 0; q < n; q++) {
                uint32_t ux = NODE(i, X_SLOT(q)), uz = NODE(i, Z_SLOT(q));
                size_t a = (size_t)(i + 1) * n + q;
                switch (kind[a]) {
                    case -1:
                        g->succ[ux] = pack2(NODE(i + 1, X_SLOT(q)), NO_SUCC);
                        g->succ[uz] = pack2(NODE(i + 1, Z_SLOT(q)), NO_SUCC);
                        break;
                    case G_H:
                        g->succ[ux] = pack2(NODE(i + 1, Z_SLOT(q)), NO_SUCC);
                        g->succ[uz] = pack2(NODE(i + 1, X_SLOT(q)), NO_SUCC);
                        break;
                    case G_CX:
                        if (ctrl[a]) {
                            g->succ[ux] = pack2(NODE(i + 1, X_SLOT(q)), NODE(i + 1, X_SLOT(partner[a])));
                            g->succ[uz] = pack2(NODE(i + 1, Z_SLOT(q)), NO_SUCC);
                        } else {
                            g->succ[ux] = pack2(NODE(i + 1, X_SLOT(q)), NO_SUCC);
                            g->succ[uz] = pack2(NODE(i + 1, Z_SLOT(partner[a])), NODE(i + 1, Z_SLOT(q)));
                        }
                        break;
                    case G_R:
                        break;
                    case G_M:
                        g->succ[ux] = pack2(LEAF((uint32_t)meas[a]), NODE(i + 1, X_SLOT(q)));
                        break;
                    case G_MR:
                        g->succ[ux] = pack2(LEAF((uint32_t)meas[a]), NO_SUCC);
                        break;
                }
            }
        }
        /* Correlated slots reference same-boundary nodes (stepg.cpp:236-254). */
        if (level != 0) {
            for (uint32_t q = 0; q < n; q++)
                g->succ[NODE(i, Y_SLOT(q))] = pack2(NODE(i, X_SLOT(q)), NODE(i, Z_SLOT(q)));
            for (uint32_t gi = c->gate_offsets[i], j = 0; gi < c->gate_offsets[i + 1]; gi++) {
                if (c->gate_kind[gi] != G_CX) continue;
                uint32_t cq = c->gate_q0[gi], tq = c->gate_q1[gi];
                g->succ[NODE(i, XZ_SLOT(j))] = pack2(NODE(i, X_SLOT(cq)), NODE(i, Z_SLOT(tq)));
                g->succ[NODE(i, ZX_SLOT(j))] = pack2(NODE(i, Z_SLOT(cq)), NODE(i, X_SLOT(tq)));
                if (level == 2) {
                    g->succ[NODE(i, XY_SLOT(j))] = pack2(NODE(i, X_SLOT(cq)), NODE(i, Y_SLOT(tq)));
                    g->succ[NODE(i, YX_SLOT(j))] = pack2(NODE(i, Y_SLOT(cq)), NODE(i, X_SLOT(tq)));
                    g->succ[NODE(i, YY_SLOT(j))] = pack2(NODE(i, Y_SLOT(cq)), NODE(i, Y_SLOT(tq)));
                    g->succ[NODE(i, YZ_SLOT(j))] = pack2(NODE(i, Y_SLOT(cq)), NODE(i, Z_SLOT(tq)));
                    g->succ[NODE(i, ZY_SLOT(j))] = pack2(NODE(i, Z_SLOT(cq)), NODE(i, Y_SLOT(tq)));
                }
                j++;
            }
        }
    }

    /* Map semantic sources onto graph nodes (stepg.cpp:257-313). */
    specs_t specs = {0};
    if (!enumerate_sources(c, level, &specs)) return fail(4, "out of memory");
    g->src = malloc((specs.n + 1) * sizeof(source_t));
    if (!g->src) return fail(4, "out of memory");
    for (size_t si = 0; si < specs.n; si++) {
        const spec_t *s = &specs.v[si];
        source_t *o = &g->src[si];
        o->prob = s->prob;
        o->node1 = NO_SUCC;
        if (s->measurement >= 0) {
            o->node0 = LEAF((uint32_t)s->measurement);
            continue;
        }
        uint32_t b = (uint32_t)s->boundary;
#define TERM(t) \
    (s->p[t] == P_X ? NODE(b, X_SLOT(s->q[t])) : s->p[t] == P_Z ? NODE(b, Z_SLOT(s->q[t])) : NODE(b, Y_SLOT(s->q[t])))
        if (s->nterms == 1) {
            o->node0 = TERM(0);
            continue;
        }
        /* Dedicated per-CX slot when (q0, q1) is a CX of layer b. */
        size_t a = (size_t)b * n + s->q[0];
        if (cxj[a] >= 0 && partner[a] == s->q[1]) {
            uint32_t j = (uint32_t)cxj[a];
            uint8_t pa = s->p[0], pb = s->p[1];
            uint32_t slot = NO_SUCC;
            if (level != 0) {
                if (pa == P_X && pb == P_Z) slot = XZ_SLOT(j);
                else if (pa == P_Z && pb == P_X) slot = ZX_SLOT(j);
            }
            if (level == 2 && slot == NO_SUCC) {
                if (pa == P_X && pb == P_Y) slot = XY_SLOT(j);
                else if (pa == P_Y && pb == P_X) slot = YX_SLOT(j);
                else if (pa == P_Y && pb == P_Y) slot = YY_SLOT(j);
                else if (pa == P_Y && pb == P_Z) slot = YZ_SLOT(j);
                else if (pa == P_Z && pb == P_Y) slot = ZY_SLOT(j);
            }
            if (slot != NO_SUCC) {
                o->node0 = NODE(b, slot);
                continue;
            }
        }
        o->node0 = TERM(0);
        o->node1 = TERM(1);
#undef TERM
    }
    g->S = specs.n;
    free(specs.v);
    free(kind);
    free(partner);
    free(ctrl);
    free(meas);
    free(cxj);
    return 0;
#undef NODE
#undef LEAF
}

/* ---- class matrix + Alg. 1: eec.cpp:22-140 --------------------------- */

typedef struct {
    uint32_t rows, W;
    uint64_t *st; /* column-major: addr = w * rows + u (eec.hpp:28-50) */
} eec_t;

#define WORD(m, u, w) ((m)->st[(size_t)(w) * (m)->rows + (u)])

/* EecMatrix::zeroed (eec.cpp:22-30) + init_leaves (eec.cpp:40-58). */
static int init_matrix(const oracle_circuit *c, const stepg_t *g, eec_t *m) {
    m->rows = g->l * g->k + g->M;
    m->W = (g->D + g->O + 63) / 64;
    m->st = calloc((size_t)m->W * m->rows + 1, sizeof(uint64_t));
    if (!m->st) return fail(4, "out of memory");
    for (uint32_t d = 0; d < g->D; d++)
        for (uint32_t t = c->det_offsets[d]; t < c->det_offsets[d + 1]; t++) {
            uint32_t me = c->det_meas[t];
            if (me >= g->M) return fail(2, "detector references a measurement without a leaf");
            WORD(m, g->l * g->k + me, d >> 6) ^= 1ull << (d & 63);
        }
    for (uint32_t o = 0; o < g->O; o++)
        for (uint32_t t = c->obs_offsets[o]; t < c->obs_offsets[o + 1]; t++) {
            uint32_t me = c->obs_meas[t];
            if (me >= g->M) return fail(3, "observable references a measurement without a leaf");
            uint32_t b = g->D + o;
            WORD(m, g->l * g->k + me, b >> 6) ^= 1ull << (b & 63);
        }
    return 0;
}

/* update_cell / run_subpass / run_backward (eec.cpp:64-122), serial schedule. */
static void run_subpass(const stepg_t *g, eec_t *m, uint32_t i, uint32_t s0, uint32_t s1) {
    for (uint32_t s = s0; s < s1; s++) {
        uint32_t u = i * g->k + s;
        uint32_t v0 = (uint32_t)g->succ[u], v1 = (uint32_t)(g->succ[u] >> 32);
        for (uint32_t w = 0; w < m->W; w++) {
            uint64_t acc = 0;
            if (v0 != NO_SUCC) acc ^= WORD(m, v0, w);
            if (v1 != NO_SUCC) acc ^= WORD(m, v1, w);
            WORD(m, u, w) = acc;
        }
    }
}

static void run_backward(const stepg_t *g, eec_t *m) {
    const uint32_t n = g->n;
    for (uint32_t i = g->l; i-- > 0;) {
        run_subpass(g, m, i, 0, 2 * n);
        if (g->level != 0) run_subpass(g, m, i, 2 * n, 4 * n);
        if (g->level == 2) run_subpass(g, m, i, 4 * n, 7 * n);
    }
}

/* ---- reduce: dem.cpp:57-142 ------------------------------------------ */

typedef struct {
    const uint64_t *sig;
    const uint64_t *keys;
    uint32_t W;
} sortctx_t;

static int cmp_words(const uint64_t *a, const uint64_t *b, uint32_t W) {
    for (uint32_t w = 0; w < W; w++)
        if (a[w] != b[w]) return a[w] < b[w] ? -1 : 1;
    return 0;
}

/* (key, lexicographic words) order, dem.cpp:73-78. */
static int cmp_key_sig(const void *pa, const void *pb, void *vctx) {
    const sortctx_t *x = vctx;
    uint32_t a = *(const uint32_t *)pa, b = *(const uint32_t *)pb;
    if (x->keys[a] != x->keys[b]) return x->keys[a] < x->keys[b] ? -1 : 1;
    int c = cmp_words(x->sig + (size_t)a * x->W, x->sig + (size_t)b * x->W, x->W);
    if (c) return c;
    return a < b ? -1 : a > b;
}

static int cmp_double(const void *pa, const void *pb) {
    double a = *(const double *)pa, b = *(const double *)pb;
    return a < b ? -1 : a > b;
}

static int cmp_u32(const void *pa, const void *pb) {
    uint32_t a = *(const uint32_t *)pa, b = *(const uint32_t *)pb;
    return a < b ? -1 : a > b;
}

typedef struct {
    uint32_t *dets, nd, *obs, no;
    double p;
    uint32_t *mem, nm;
} group_t;

/* std::vector<uint32_t> lexicographic compare (prefix sorts first). */
static int cmp_list(const uint32_t *a, uint32_t na, const uint32_t *b, uint32_t nb) {
    uint32_t m = na < nb ? na : nb;
    for (uint32_t i = 0; i < m; i++)
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return na < nb ? -1 : na > nb;
}

/* Canonical order (dem.cpp:122-127): detectors first, then observables. */
static int cmp_group(const void *pa, const void *pb) {
    const group_t *a = pa, *b = pb;
    int c = cmp_list(a->dets, a->nd, b->dets, b->nd);
    if (c) return c;
    return cmp_list(a->obs, a->no, b->obs, b->no);
}

static int reduce_packed(const uint64_t *sig, const double *probs, size_t count, uint32_t W,
                         uint32_t D, uint32_t O, oracle_dem *out) {
    uint64_t *keys = malloc((count + 1) * sizeof(uint64_t));
    uint32_t *order = malloc((count + 1) * sizeof(uint32_t));
    group_t *groups = malloc((count + 1) * sizeof(group_t));
    double *fold = malloc((count + 1) * sizeof(double));
    if (!keys || !order || !groups || !fold) return fail(4, "out of memory");
    for (size_t i = 0; i < count; i++) {
        keys[i] = oracle_fnv1_64(sig + i * W, W); /* dem.cpp:61-64 */
        order[i] = (uint32_t)i;
    }
    sortctx_t ctx = {sig, keys, W};
    qsort_r(order, count, sizeof(uint32_t), cmp_key_sig, &ctx);
    size_t ng = 0, i = 0;
    while (i < count) { /* group scan, dem.cpp:87-121 */
        size_t j = i;
        const uint64_t *s = sig + (size_t)order[i] * W;
        while (j < count && cmp_words(sig + (size_t)order[j] * W, s, W) == 0) j++;
        int empty = 1;
        for (uint32_t w = 0; w < W; w++)
            if (s[w]) empty = 0;
        if (!empty) {
            group_t *g = &groups[ng++];
            size_t nf = 0;
            g->nm = (uint32_t)(j - i);
            g->mem = malloc(g->nm * sizeof(uint32_t));
            for (size_t t = i; t < j; t++) {
                fold[nf++] = probs[order[t]];
                g->mem[t - i] = order[t];
            }
            qsort(fold, nf, sizeof(double), cmp_double); /* canonical fold order */
            double p = 0;
            for (size_t t = 0; t < nf; t++) p = oracle_merge_prob(p, fold[t]);
            g->p = p;
            g->dets = malloc((D + O + 1) * sizeof(uint32_t));
            g->obs = malloc((O + 1) * sizeof(uint32_t));
            g->nd = g->no = 0;
            for (uint32_t b = 0; b < D + O; b++)
                if (s[b >> 6] >> (b & 63) & 1) {
                    if (b < D) g->dets[g->nd++] = b;
                    else g->obs[g->no++] = b - D;
                }
            qsort(g->mem, g->nm, sizeof(uint32_t), cmp_u32);
        }
        i = j;
    }
    qsort(groups, ng, sizeof(group_t), cmp_group);

    out->num_detectors = D;
    out->num_observables = O;
    out->num_edges = ng;
    out->det_offsets = malloc((ng + 1) * sizeof(uint64_t));
    out->obs_offsets = malloc((ng + 1) * sizeof(uint64_t));
    out->mem_offsets = malloc((ng + 1) * sizeof(uint64_t));
    out->probs = malloc((ng + 1) * sizeof(double));
    size_t td = 0, to = 0, tm = 0;
    for (size_t e = 0; e < ng; e++) {
        td += groups[e].nd;
        to += groups[e].no;
        tm += groups[e].nm;
    }
    out->det_ids = malloc((td + 1) * sizeof(uint32_t));
    out->obs_ids = malloc((to + 1) * sizeof(uint32_t));
    out->mem_ids = malloc((tm + 1) * sizeof(uint32_t));
    td = to = tm = 0;
    for (size_t e = 0; e < ng; e++) {
        group_t *g = &groups[e];
        out->det_offsets[e] = td;
        out->obs_offsets[e] = to;
        out->mem_offsets[e] = tm;
        memcpy(out->det_ids + td, g->dets, g->nd * sizeof(uint32_t));
        memcpy(out->obs_ids + to, g->obs, g->no * sizeof(uint32_t));
        memcpy(out->mem_ids + tm, g->mem, g->nm * sizeof(uint32_t));
        td += g->nd;
        to += g->no;
        tm += g->nm;
        out->probs[e] = g->p;
        free(g->dets);
        free(g->obs);
        free(g->mem);
    }
    out->det_offsets[ng] = td;
    out->obs_offsets[ng] = to;
    out->mem_offsets[ng] = tm;
    free(keys);
    free(order);
    free(groups);
    free(fold);
    return 0;
}

/* compile_circuit (compile.cpp:23-53). */
int oracle_compile(const oracle_circuit *c, int level, oracle_dem *out) {
    memset(out, 0, sizeof *out);
    stepg_t g;
    int rc = lower(c, level, &g);
    if (rc) return rc;
    eec_t m;
    rc = init_matrix(c, &g, &m);
    if (rc) {
        free(g.succ);
        free(g.src);
        return rc;
    }
    run_backward(&g, &m);
    /* Dense signature gather (compile.cpp:34-39 -> eec.cpp:130-140). */
    uint64_t *sig = malloc(((size_t)g.S * m.W + 1) * sizeof(uint64_t));
    double *probs = malloc((g.S + 1) * sizeof(double));
    if (!sig || !probs) return fail(4, "out of memory");
    for (size_t s = 0; s < g.S; s++) {
        for (uint32_t w = 0; w < m.W; w++) {
            uint64_t acc = WORD(&m, g.src[s].node0, w);
            if (g.src[s].node1 != NO_SUCC) acc ^= WORD(&m, g.src[s].node1, w);
            sig[s * m.W + w] = acc;
        }
        probs[s] = g.src[s].prob;
    }
    rc = reduce_packed(sig, probs, g.S, m.W, g.D, g.O, out);
    out->num_sources = g.S;
    free(sig);
    free(probs);
    free(m.st);
    free(g.succ);
    free(g.src);
    return rc;
}

/* ---- forward oracle: frame.cpp:159-239 -------------------------------- */

/* FrameSim::apply_gates with collapse randomisation off (frame.cpp:59-90). */
static void apply_gates(const oracle_circuit *c, uint32_t layer, uint8_t *x, uint8_t *z,
                        uint8_t *meas) {
    for (uint32_t g = c->gate_offsets[layer]; g < c->gate_offsets[layer + 1]; g++) {
        uint32_t q0 = c->gate_q0[g], q1 = c->gate_q1[g];
        uint8_t t;
        switch (c->gate_kind[g]) {
            case G_H:
                t = x[q0];
                x[q0] = z[q0];
                z[q0] = t;
                break;
            case G_CX:
                x[q1] ^= x[q0];
                z[q0] ^= z[q1];
                break;
            case G_R:
                x[q0] = 0;
                z[q0] = 0;
                break;
            case G_M:
                meas[c->gate_meas[g]] ^= x[q0];
                z[q0] = 0;
                break;
            case G_MR:
                meas[c->gate_meas[g]] ^= x[q0];
                x[q0] = 0;
                z[q0] = 0;
                break;
        }
    }
}

int oracle_forward(const oracle_circuit *c, int level, oracle_dem *out) {
    memset(out, 0, sizeof *out);
    specs_t specs = {0};
    if (!enumerate_sources(c, level, &specs)) return fail(4, "out of memory");
    const uint32_t D = c->num_detectors, O = c->num_observables, W = (D + O + 63) / 64;
    uint64_t *sig = calloc((size_t)specs.n * W + 1, sizeof(uint64_t));
    double *probs = malloc((specs.n + 1) * sizeof(double));
    uint8_t *x = malloc(c->num_qubits + 1), *z = malloc(c->num_qubits + 1);
    uint8_t *meas = malloc(c->num_measurements + 1);
    if (!sig || !probs || !x || !z || !meas) return fail(4, "out of memory");
    for (size_t si = 0; si < specs.n; si++) { /* propagate_error */
        const spec_t *s = &specs.v[si];
        memset(x, 0, c->num_qubits);
        memset(z, 0, c->num_qubits);
        memset(meas, 0, c->num_measurements);
        if (s->measurement >= 0) {
            meas[s->measurement] ^= 1;
        } else {
            for (uint32_t t = 0; t < s->nterms; t++) { /* apply_pauli, frame.cpp:50-57 */
                if (s->p[t] != P_Z) x[s->q[t]] ^= 1;
                if (s->p[t] != P_X) z[s->q[t]] ^= 1;
            }
            for (uint32_t i = (uint32_t)s->boundary + 1; i < c->num_layers; i++)
                apply_gates(c, i, x, z, meas);
        }
        uint64_t *row = sig + si * W;
        for (uint32_t d = 0; d < D; d++) {
            uint8_t v = 0;
            for (uint32_t t = c->det_offsets[d]; t < c->det_offsets[d + 1]; t++) v ^= meas[c->det_meas[t]];
            if (v) row[d >> 6] |= 1ull << (d & 63);
        }
        for (uint32_t o = 0; o < O; o++) {
            uint8_t v = 0;
            for (uint32_t t = c->obs_offsets[o]; t < c->obs_offsets[o + 1]; t++) v ^= meas[c->obs_meas[t]];
            uint32_t b = D + o;
            if (v) row[b >> 6] |= 1ull << (b & 63);
        }
        probs[si] = s->prob;
    }
    /* build_dem_oracle groups by exact signature (std::map) and applies the
     * same sorted fold and canonical order; reduce_packed is equivalent. */
    int rc = reduce_packed(sig, probs, specs.n, W, D, O, out);
    out->num_sources = specs.n;
    free(specs.v);
    free(sig);
    free(probs);
    free(x);
    free(z);
    free(meas);
    return rc;
}

void oracle_dem_free(oracle_dem *d) {
    free(d->det_offsets);
    free(d->det_ids);
    free(d->obs_offsets);
    free(d->obs_ids);
    free(d->probs);
    free(d->mem_offsets);
    free(d->mem_ids);
    memset(d, 0, sizeof *d);
}

// gp_api.cpp -- C ABI (include/greenpeas.h) of the B200 DEM compiler.
//
// gp_compile / gp_compile_batch replace demc::compile_circuit
// (/root/reference/proj/core/src/compile.cpp:23-53). The host side does only
// what cannot run on the GPU: it validates the reference's error conditions,
// packs the flat circuit view into one pinned staging image (compact 8/16-byte
// op words), uploads it with one async copy, enqueues the device pipeline
// (gp_kernels.cu) and downloads the flat DEM into context-owned pinned memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <charconv>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/greenpeas.h"
#include "gp_device.h"
#include "gp_layout.h"

using gp::BatchTotals;
using gp::CircuitMeta;
using gp::DevPlan;
using gp::DeviceHeader;
using gp::StageLayout;

// Per-circuit counts of pass 1 (independent across circuits).
struct CircCount {
    int err;  // 0 ok, 1 index space, 2 detector leaf, 3 observable leaf, 4 too wide
    uint32_t src_noise, max_noise, max_meas;
    uint64_t gates, noise, det_entries, obs_entries;
    std::vector<double> probs;  // distinct noise probabilities (<= kLocalProbs, else many)
    std::vector<uint32_t> pidx; // global table index of each local probability
    bool many;
};
constexpr size_t kLocalProbs = 64;

struct gp_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    int force_collisions = 0;
    uint32_t trav_debug = 0;
    uint32_t record_slots = 8;
    uint64_t ids_hint = 0;  // learned id capacity (grows on overflow)
    uint64_t pool_hint = 0; // learned record-pool chunks (grows on overflow)

    uint8_t *h_stage = nullptr;
    size_t h_stage_cap = 0;
    uint8_t *d_img = nullptr;
    size_t d_img_cap = 0;
    uint8_t *d_ws = nullptr;
    size_t d_ws_cap = 0;
    uint8_t *h_out = nullptr;
    size_t h_out_cap = 0;
    DeviceHeader *h_hdr = nullptr;

    cudaEvent_t ev_start = nullptr, ev_h2d = nullptr, ev_end = nullptr;
    gp::StageEvents stage_ev{};

    std::vector<CircuitMeta> metas;
    std::vector<uint32_t> out_ndet, out_nobs;
    std::vector<double> prob_table;
    std::vector<CircCount> circ_counts;

    // Last successful device plan (for gp_replay) and profiling state.
    bool has_plan = false;
    DevPlan last_plan{};
    cudaEvent_t prof[gp::kProfCount] = {};
    uint64_t prof_ns[gp::kProfCount] = {};
    uint8_t *d_flush = nullptr;
    uint64_t *d_dbg = nullptr;  // experiments only (option 99, bit 2)
};

namespace {

using clk = std::chrono::steady_clock;

uint64_t ns_since(clk::time_point t0) {
    return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(clk::now() - t0).count();
}

uint64_t align16(uint64_t x) { return (x + 15) & ~15ull; }

gp_status fail(gp_ctx *ctx, gp_status st, const std::string &msg) {
    ctx->err = msg;
    return st;
}

gp_status cuda_fail(gp_ctx *ctx, cudaError_t e, const char *what) {
    return fail(ctx, GP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

uint32_t alpha_of(uint8_t level) { return level == 0 ? 2 : level == 1 ? 4 : 7; }  // stepg.cpp:23-33

uint32_t components(uint8_t kind, uint8_t level) {  // stepg.cpp:66-103
    if (kind <= GP_NOISE_Z_ERROR) return 1;
    if (kind == GP_NOISE_DEPOLARIZE1) return level == 0 ? 2 : 3;
    return level == 0 ? 6 : level == 1 ? 10 : 15;
}

// Runs f(i) for i in [0, n) on up to hardware_concurrency host threads
// (inline for small n: single-circuit latency pays no thread start-up).
template <class F>
void parallel_for(size_t n, F f) {
    const size_t hw = std::max<unsigned>(1, std::thread::hardware_concurrency());
    const size_t nt = std::min(hw, n / 32);
    if (nt <= 1) {
        for (size_t i = 0; i < n; i++) f(i);
        return;
    }
    std::atomic<size_t> next{0};
    auto work = [&] {
        for (size_t i0; (i0 = next.fetch_add(16)) < n;)
            for (size_t i = i0; i < std::min(n, i0 + 16); i++) f(i);
    };
    std::vector<std::thread> pool;
    for (size_t t = 1; t < nt; t++) pool.emplace_back(work);
    work();
    for (auto &th : pool) th.join();
}



// Pass 1: validation (the reference's exceptions, in the reference's order;
// for a batch, the first failing circuit), device-encoding limits, totals and
// per-circuit metadata. Counting runs in parallel over circuits.
gp_status plan_batch(gp_ctx *ctx, const gp_circuit_view *cs, size_t C, uint8_t level, BatchTotals &t,
                     std::vector<CircuitMeta> &metas) {
    t = BatchTotals{};
    t.C = (uint32_t)C;
    t.level = level;
    metas.assign(C, CircuitMeta{});
    std::vector<CircCount> cc(C);
    parallel_for(C, [&](size_t c) {
        const gp_circuit_view &v = cs[c];
        CircCount &k = cc[c];
        k = CircCount{};
        const uint64_t rows = (uint64_t)v.num_layers * alpha_of(level) * v.num_qubits + v.num_measurements;
        if (rows >= 0xFFFFFFFFull) {  // lower(), stepg.cpp:171-174
            k.err = 1;
            return;
        }
        for (uint32_t d = 0; d < v.num_detectors; d++)  // init_leaves, eec.cpp:42-49
            for (uint32_t x = v.det_offsets[d]; x < v.det_offsets[d + 1]; x++)
                if (v.det_meas[x] >= v.num_measurements) {
                    k.err = 2;
                    return;
                }
        for (uint32_t o = 0; o < v.num_observables; o++)  // eec.cpp:50-57
            for (uint32_t x = v.obs_offsets[o]; x < v.obs_offsets[o + 1]; x++)
                if (v.obs_meas[x] >= v.num_measurements) {
                    k.err = 3;
                    return;
                }
        if (v.num_qubits >= (1u << gp::kNoiseQubitBits) || v.num_measurements >= 0x7FFFFFFFu) {
            k.err = 4;
            return;
        }
        uint64_t src = 0;
        for (uint32_t i = 0; i < v.num_layers; i++) {
            const uint32_t n0 = v.noise_offsets[i], n1 = v.noise_offsets[i + 1];
            k.max_noise = std::max(k.max_noise, n1 - n0);
            for (uint32_t o = n0; o < n1; o++) {
                src += components(v.noise_kind[o], level);
                if (k.many) continue;
                const double pr = v.noise_prob[o];
                bool seen = false;
                for (double q : k.probs) seen |= std::memcmp(&q, &pr, 8) == 0;
                if (!seen) {
                    if (k.probs.size() == kLocalProbs) k.many = true;
                    else k.probs.push_back(pr);
                }
            }
            uint32_t meas = 0;
            for (uint32_t g = v.gate_offsets[i]; g < v.gate_offsets[i + 1]; g++)
                meas += v.gate_kind[g] == GP_GATE_M || v.gate_kind[g] == GP_GATE_MR;
            k.max_meas = std::max(k.max_meas, meas);
        }
        k.src_noise = (uint32_t)src;
        k.gates = v.gate_offsets[v.num_layers] - v.gate_offsets[0];
        k.noise = v.noise_offsets[v.num_layers] - v.noise_offsets[0];
        k.det_entries = v.det_offsets[v.num_detectors] - v.det_offsets[0];
        k.obs_entries = v.obs_offsets[v.num_observables] - v.obs_offsets[0];
    });
    // Batch probability table (bit-exact keys); wide mode if it would not fit.
    {
        std::vector<uint64_t> keys;
        bool many = false;
        for (const CircCount &k : cc) {
            many |= k.many;
            for (double q : k.probs) {
                uint64_t b;
                std::memcpy(&b, &q, 8);
                keys.push_back(b);
            }
        }
        std::sort(keys.begin(), keys.end());
        keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
        t.wide_prob = many || keys.size() > gp::kNoisePidxMax;
        ctx->prob_table.clear();
        if (!t.wide_prob) {
            for (uint64_t b : keys) {
                double q;
                std::memcpy(&q, &b, 8);
                ctx->prob_table.push_back(q);
            }
            for (CircCount &k : cc) {
                k.pidx.clear();
                for (double q : k.probs) {
                    uint64_t b;
                    std::memcpy(&b, &q, 8);
                    k.pidx.push_back((uint32_t)(std::lower_bound(keys.begin(), keys.end(), b) - keys.begin()));
                }
            }
        }
        t.prob_table_n = (uint32_t)ctx->prob_table.size();
        ctx->circ_counts = std::move(cc);
    }
    std::vector<CircCount> &cc2 = ctx->circ_counts;
    static const char *kErr[] = {"", "circuit exceeds 32-bit node index space",
                                 "detector references a measurement without a leaf",
                                 "observable references a measurement without a leaf",
                                 "circuit too wide for the device encoding"};
    for (size_t c = 0; c < C; c++)
        if (cc2[c].err) return fail(ctx, cc2[c].err == 4 ? GP_ERR_UNSUPPORTED : GP_ERR_INVALID_ARGUMENT, kErr[cc2[c].err]);
    for (size_t c = 0; c < C; c++) {  // prefix sums (serial, O(C))
        const gp_circuit_view &v = cs[c];
        const CircCount &k = cc2[c];
        CircuitMeta &m = metas[c];
        m.n = v.num_qubits;
        m.l = v.num_layers;
        m.M = v.num_measurements;
        m.D = v.num_detectors;
        m.O = v.num_observables;
        m.W = (uint32_t)(((uint64_t)m.D + m.O + 63) / 64);
        m.layer_base = (uint32_t)t.layer_slots;
        m.meas_base = (uint32_t)t.meas;
        m.det_base = (uint32_t)t.det_slots;
        m.obs_base = (uint32_t)t.obs_slots;
        m.tile_base = (uint32_t)t.tiles;
        m.bucket_base = (uint32_t)t.buckets;
        m.src_base = t.sources;
        m.ell_base = t.ell;
        m.leaf_base = t.leaf;
        m.src_noise = k.src_noise;
        m.max_layer_noise = k.max_noise;
        m.gate_base = t.gates;
        m.noise_base = t.noise;
        m.det_entry_base = t.det_entries;
        m.obs_entry_base = t.obs_entries;
        m.circ_layer_base = t.layers;
        t.max_layer_noise = std::max(t.max_layer_noise, k.max_noise);
        t.max_layer_meas = std::max(t.max_layer_meas, k.max_meas);
        t.max_n = std::max(t.max_n, m.n);
        t.max_W = std::max(t.max_W, m.W);
        t.max_l = std::max(t.max_l, m.l);
        t.layers += m.l;
        t.layer_slots += m.l + 1;
        t.gates += k.gates;
        t.noise += k.noise;
        t.meas += m.M;
        t.det_slots += m.D + 1;
        t.det_entries += k.det_entries;
        t.obs_slots += m.O + 1;
        t.obs_entries += k.obs_entries;
        t.dets += m.D;
        t.obss += m.O;
        t.tiles += m.W;
        t.sources += k.src_noise + m.M;
        t.ell += m.l ? (uint64_t)(m.l - 1) * gp::ell_stride(m.n) : 0;
        t.leaf += (uint64_t)m.W * gp::leaf_stride(m.M);
        t.buckets += (uint64_t)m.D + 1;
    }
    if (t.sources >= 0xFFFFFFFFull || t.tiles >= 0xFFFFFFFFull || t.gates >= 0xFFFFFFFFull ||
        t.noise >= 0xFFFFFFFFull || t.meas >= 0xFFFFFFFFull || t.layer_slots >= 0xFFFFFFFFull)
        return fail(ctx, GP_ERR_UNSUPPORTED, "batch exceeds 32-bit device indexing; split it");
    return GP_OK;
}

StageLayout stage_layout(const BatchTotals &t) {
    StageLayout L{};
    uint64_t o = 0;
    auto put = [&](uint64_t bytes) {
        const uint64_t at = o;
        o = align16(o + bytes + 16);  // +16: bulk copies may over-read one 16-byte unit
        return at;
    };
    L.meta = put(t.C * sizeof(CircuitMeta));
    L.circ_layer = put((t.C + 1) * 4);
    L.circ_src = put((t.C + 1) * 8);
    L.circ_tile = put((t.C + 1) * 4);
    L.circ_grp = put((t.C + 1) * 4);
    L.circ_det = put((t.C + 1) * 4);
    L.circ_obs = put((t.C + 1) * 4);
    L.lay_gate = put(t.layer_slots * 4);
    L.lay_noise = put(t.layer_slots * 4);
    L.lay_meas = put(t.layer_slots * 4);
    L.gates = put(t.gates * 8);
    L.noise = put(t.noise * 8);
    L.noise_prob = put(t.wide_prob ? t.noise * 8 : 0);
    L.prob_table = put((uint64_t)t.prob_table_n * 8);
    L.lay_src = put(t.layer_slots * 4);
    L.meas_flip = put(t.meas * 8);
    L.det_off = put(t.det_slots * 4);
    L.det_meas = put(t.det_entries * 4);
    L.obs_off = put(t.obs_slots * 4);
    L.obs_meas = put(t.obs_entries * 4);
    L.total = o;
    return L;
}

// Pass 2: write the staging image, in parallel over circuits (each circuit's
// slices of every array are disjoint and located by its prefix bases).
// Cumulative per-circuit tables (O(C), serial).
void pack_tables(const BatchTotals &t, const std::vector<CircuitMeta> &metas, const StageLayout &L, uint32_t T,
                 const std::vector<double> &ptab, uint8_t *img) {
    auto at = [&](uint64_t off) { return img + off; };
    if (!ptab.empty()) std::memcpy(at(L.prob_table), ptab.data(), ptab.size() * 8);
    std::memcpy(at(L.meta), metas.data(), t.C * sizeof(CircuitMeta));
    auto *circ_layer = (uint32_t *)at(L.circ_layer);
    auto *circ_src = (uint64_t *)at(L.circ_src);
    auto *circ_tile = (uint32_t *)at(L.circ_tile);
    auto *circ_grp = (uint32_t *)at(L.circ_grp);
    auto *circ_det = (uint32_t *)at(L.circ_det);
    auto *circ_obs = (uint32_t *)at(L.circ_obs);
    uint64_t grps = 0, dets = 0, obss = 0;
    for (uint32_t c = 0; c < t.C; c++) {  // O(C) cumulative tables
        const CircuitMeta &m = metas[c];
        circ_layer[c] = (uint32_t)m.circ_layer_base;
        circ_src[c] = m.src_base;
        circ_tile[c] = m.tile_base;
        circ_grp[c] = (uint32_t)grps;
        circ_det[c] = (uint32_t)dets;
        circ_obs[c] = (uint32_t)obss;
        grps += (m.W + T - 1) / T;
        dets += m.D;
        obss += m.O;
    }
    circ_layer[t.C] = (uint32_t)t.layers;
    circ_src[t.C] = t.sources;
    circ_tile[t.C] = (uint32_t)t.tiles;
    circ_grp[t.C] = (uint32_t)grps;
    circ_det[t.C] = (uint32_t)dets;
    circ_obs[t.C] = (uint32_t)obss;
}

// Per-circuit slices of every section for circuits [c0, c1), in parallel.
void pack_circuits(const gp_circuit_view *cs, const BatchTotals &t, const std::vector<CircuitMeta> &metas,
                   const std::vector<CircCount> &cc, const StageLayout &L, uint8_t *img, size_t c0, size_t c1) {
    auto at = [&](uint64_t off) { return img + off; };
    auto *lay_gate = (uint32_t *)at(L.lay_gate);
    auto *lay_noise = (uint32_t *)at(L.lay_noise);
    auto *lay_meas = (uint32_t *)at(L.lay_meas);
    auto *gates = (uint64_t *)at(L.gates);
    auto *noise = (uint64_t *)at(L.noise);
    auto *nprob = (double *)at(L.noise_prob);
    auto *lay_src = (uint32_t *)at(L.lay_src);
    auto *flip = (double *)at(L.meas_flip);
    auto *det_off = (uint32_t *)at(L.det_off);
    auto *det_meas = (uint32_t *)at(L.det_meas);
    auto *obs_off = (uint32_t *)at(L.obs_off);
    auto *obs_meas = (uint32_t *)at(L.obs_meas);
    parallel_for(c1 - c0, [&](size_t ci) {
        const size_t c = c0 + ci;
        const gp_circuit_view &v = cs[c];
        const CircuitMeta &m = metas[c];
        const uint64_t g_at = m.gate_base, n_at = m.noise_base;
        const uint32_t g0 = v.gate_offsets[0], n0 = v.noise_offsets[0];
        uint32_t src = 0, meas = 0;
        for (uint32_t i = 0; i <= m.l; i++) {
            lay_gate[m.layer_base + i] = (uint32_t)(g_at + v.gate_offsets[i] - g0);
            lay_noise[m.layer_base + i] = (uint32_t)(n_at + v.noise_offsets[i] - n0);
            lay_meas[m.layer_base + i] = meas;
            lay_src[m.layer_base + i] = src;
            if (i == m.l) break;
            for (uint32_t g = v.gate_offsets[i]; g < v.gate_offsets[i + 1]; g++) {
                const uint8_t k = v.gate_kind[g];
                uint32_t hi = 0;
                if (k == GP_GATE_CX) hi = v.gate_q1[g];
                if (k == GP_GATE_M || k == GP_GATE_MR) {
                    hi = (uint32_t)v.gate_meas[g];
                    flip[m.meas_base + hi] = v.gate_flip[g];
                    meas++;
                }
                gates[g_at + g - g0] = (uint64_t)hi << 32 | (v.gate_q0[g] | (uint32_t)k << gp::kGateKindShift);
            }
            const CircCount &k2 = cc[c];
            for (uint32_t o = v.noise_offsets[i]; o < v.noise_offsets[i + 1]; o++) {
                const uint8_t k = v.noise_kind[o];
                const uint64_t idx = n_at + o - n0;
                uint64_t pidx = 0;
                const double pr = v.noise_prob[o];
                if (t.wide_prob) {
                    nprob[idx] = pr;
                } else {
                    for (size_t x = 0; x < k2.probs.size(); x++)
                        if (std::memcmp(&k2.probs[x], &pr, 8) == 0) {
                            pidx = k2.pidx[x];
                            break;
                        }
                }
                noise[idx] = (uint64_t)v.noise_q0[o] |
                             (uint64_t)(k == GP_NOISE_DEPOLARIZE2 ? v.noise_q1[o] : 0) << gp::kNoiseQubitBits |
                             (uint64_t)k << gp::kNoiseKindShift | pidx << gp::kNoisePidxShift;
                src += components(k, (uint8_t)t.level);
            }
        }
        const uint64_t de_at = m.det_entry_base, oe_at = m.obs_entry_base;
        for (uint32_t d = 0; d <= m.D; d++)
            det_off[m.det_base + d] = (uint32_t)(de_at + v.det_offsets[d] - v.det_offsets[0]);
        const uint32_t nde = v.det_offsets[m.D] - v.det_offsets[0];
        if (nde) std::memcpy(det_meas + de_at, v.det_meas + v.det_offsets[0], nde * 4);
        for (uint32_t o = 0; o <= m.O; o++)
            obs_off[m.obs_base + o] = (uint32_t)(oe_at + v.obs_offsets[o] - v.obs_offsets[0]);
        const uint32_t noe = v.obs_offsets[m.O] - v.obs_offsets[0];
        if (noe) std::memcpy(obs_meas + oe_at, v.obs_meas + v.obs_offsets[0], noe * 4);
    });
}

// Device workspace carve-up for a batch (capacity-checked, grown on demand).
struct WsPlan {
    size_t bytes = 0;
    uint64_t table_cap = 0, bsum_cap = 0, ids_cap = 0;
    struct Slot {
        void **dst;
        size_t bytes;
    };
};

size_t carve(gp_ctx *ctx, DevPlan &p, const BatchTotals &t, uint8_t *base, uint32_t K, uint64_t ids_cap,
             uint64_t pool_chunks, uint64_t slabs) {
    const uint64_t S = t.sources;
    uint64_t cap = 1024;
    while (cap < S + S / 2 + 16) cap <<= 1;
    const uint64_t nb = std::max<uint64_t>(S, t.buckets + 1) / 2048 + 16;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o = (size_t)align16(o + bytes + 16);
        return base ? base + at : nullptr;
    };
    p.ell = (uint32_t *)take(t.ell * 4);
    p.leaf = (uint64_t *)take(t.leaf * 8);
    p.prob = (double *)take(S * 8);
    p.nsrc = (uint32_t *)take(t.noise * 4 + 16);
    p.cnt = (uint32_t *)take(S * 4 + 4);
    p.rbits = (uint64_t *)take(S * K * 8);
    p.rtile = (uint32_t *)take(S * K * 4);
    p.K = K;
    p.pool = (uint4 *)take(pool_chunks * gp::kPoolChunk * 16);
    p.pool_chunks_cap = (uint32_t)pool_chunks;
    p.slab_words = (2 * t.max_n + 1) & ~1u;
    p.slab_stride = slabs ? t.max_l : 0;
    p.slab = (uint64_t *)take(slabs * p.slab_words * 8);
    p.slab_hdr = (uint4 *)take(slabs * 16);
    p.rep = (uint32_t *)take(S * 4);
    p.gcnt = (uint32_t *)take(S * 4 + 4);
    p.ecnt = (uint2 *)take(S * 8);
    p.sscan = (uint4 *)take(S * 16);
    p.table = (uint64_t *)take(cap * 8);
    p.table_mask = cap - 1;
    p.force_collisions = ctx->force_collisions;
    p.e_src = (uint32_t *)take(S * 4);
    p.e_idoff = (uint32_t *)take(S * 4);
    p.e_nd = (uint32_t *)take(S * 4);
    p.e_no = (uint32_t *)take(S * 4);
    p.e_moff = (uint32_t *)take(S * 4 + 4);
    p.e_bucket = (uint32_t *)take(S * 4);
    p.e_circ = (uint32_t *)take(S * 4);
    p.blist = (uint32_t *)take(S * 4);
    p.perm = (uint32_t *)take(S * 4);
    p.e_prob = (double *)take(S * 8);
    p.mprob = (double *)take(S * 8);
    p.pscan = (uint4 *)take(S * 16 + 16);
    p.tid = (uint32_t *)take(ids_cap * 4);
    p.ids_cap = ids_cap;
    p.bcount = (uint32_t *)take(t.buckets * 4 + 4);
    p.boff = (uint4 *)take((t.buckets + 1) * 16);
    p.bsum = (uint4 *)take(nb * 16);
    p.bsum_cap = nb;
    p.o_det_off = (uint64_t *)take(S * 8 + 8);
    p.o_obs_off = (uint64_t *)take(S * 8 + 8);
    p.o_det = (uint32_t *)take(ids_cap * 4);
    p.o_obs = (uint32_t *)take(ids_cap * 4);
    p.o_prob = (double *)take(S * 8);
    p.o_edge_off = (uint64_t *)take((t.C + 1) * 8);
    p.hdr = (DeviceHeader *)take(sizeof(DeviceHeader));
    return o;
}

gp_status ensure_device(gp_ctx *ctx, uint8_t **buf, size_t *cap, size_t need) {
    if (*cap >= need) return GP_OK;
    if (*buf) cudaFree(*buf);
    *buf = nullptr;
    *cap = 0;
    size_t want = need + need / 4;
    cudaError_t e = cudaMalloc(buf, want);
    if (e != cudaSuccess) {
        cudaGetLastError();
        e = cudaMalloc(buf, need);
        want = need;
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        *buf = nullptr;
        return fail(ctx, GP_ERR_OUT_OF_MEMORY, "device allocation of " + std::to_string(need) + " bytes failed");
    }
    *cap = want;
    return GP_OK;
}

gp_status ensure_host(gp_ctx *ctx, uint8_t **buf, size_t *cap, size_t need) {
    if (*cap >= need) return GP_OK;
    if (*buf) cudaFreeHost(*buf);
    *buf = nullptr;
    *cap = 0;
    const size_t want = need + need / 4 + 4096;
    if (cudaMallocHost(buf, want) != cudaSuccess) {
        cudaGetLastError();
        *buf = nullptr;
        return fail(ctx, GP_ERR_OUT_OF_MEMORY, "pinned host allocation failed");
    }
    *cap = want;
    return GP_OK;
}

float elapsed_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return ms;
}

struct HostOut {
    uint64_t *det_off, *obs_off, *edge_off;
    double *probs;
    uint32_t *det_ids, *obs_ids;
};

gp_status run_batch(gp_ctx *ctx, const gp_circuit_view *cs, size_t count, uint8_t level, HostOut &ho,
                    DeviceHeader &hdr, gp_stats *stats) {
    const auto t0 = clk::now();
    if (level > 2) return fail(ctx, GP_ERR_INVALID_ARGUMENT, "correlation level must be 0, 1 or 2");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, GP_ERR_CUDA, "cudaSetDevice failed");
    BatchTotals t;
    gp_status st = plan_batch(ctx, cs, count, level, t, ctx->metas);
    if (st != GP_OK) return st;
    gp::TravCfg tcfg;
    size_t tsmem;
    if (!gp::plan_traversal(t, ctx->device, &tcfg, &tsmem))
        return fail(ctx, GP_ERR_UNSUPPORTED, "circuit too wide for on-chip traversal state (2n words)");
    t.groups = 0;
    for (const CircuitMeta &m : ctx->metas) t.groups += (m.W + tcfg.T - 1) / tcfg.T;
    const StageLayout L = stage_layout(t);
    if ((st = ensure_host(ctx, &ctx->h_stage, &ctx->h_stage_cap, L.total)) != GP_OK) return st;
    if ((st = ensure_device(ctx, &ctx->d_img, &ctx->d_img_cap, L.total)) != GP_OK) return st;

    // Pack in circuit chunks; each chunk's slice of every section is copied
    // while the next chunk is packed (the image is circuit-major per section).
    cudaError_t e = cudaSuccess;
    cudaEventRecord(ctx->ev_start, ctx->stream);
    const std::vector<CircuitMeta> &M = ctx->metas;
    const size_t nchunk = count >= 1024 ? 8 : count >= 256 ? 4 : 1;
    auto slice = [&](uint64_t off, uint64_t elem, uint64_t lo, uint64_t hi) {
        if (hi > lo && e == cudaSuccess)
            e = cudaMemcpyAsync(ctx->d_img + off + lo * elem, ctx->h_stage + off + lo * elem, (hi - lo) * elem,
                                cudaMemcpyHostToDevice, ctx->stream);
    };
    for (size_t k = 0; k < nchunk; k++) {
        const size_t c0 = count * k / nchunk, c1 = count * (k + 1) / nchunk;
        if (c1 == c0) continue;
        pack_circuits(cs, t, M, ctx->circ_counts, L, ctx->h_stage, c0, c1);
        const CircuitMeta &a = M[c0];
        const bool last = c1 == count;
        const CircuitMeta *b = last ? nullptr : &M[c1];
        slice(L.lay_gate, 4, a.layer_base, last ? t.layer_slots : b->layer_base);
        slice(L.lay_noise, 4, a.layer_base, last ? t.layer_slots : b->layer_base);
        slice(L.lay_meas, 4, a.layer_base, last ? t.layer_slots : b->layer_base);
        slice(L.gates, 8, a.gate_base, last ? t.gates : b->gate_base);
        slice(L.noise, 8, a.noise_base, last ? t.noise : b->noise_base);
        if (t.wide_prob) slice(L.noise_prob, 8, a.noise_base, last ? t.noise : b->noise_base);
        slice(L.lay_src, 4, a.layer_base, last ? t.layer_slots : b->layer_base);
        slice(L.meas_flip, 8, a.meas_base, last ? t.meas : b->meas_base);
        slice(L.det_off, 4, a.det_base, last ? t.det_slots : b->det_base);
        slice(L.det_meas, 4, a.det_entry_base, last ? t.det_entries : b->det_entry_base);
        slice(L.obs_off, 4, a.obs_base, last ? t.obs_slots : b->obs_base);
        slice(L.obs_meas, 4, a.obs_entry_base, last ? t.obs_entries : b->obs_entry_base);
    }
    pack_tables(t, M, L, tcfg.T, ctx->prob_table, ctx->h_stage);
    slice(0, 1, 0, L.lay_gate);  // meta + cumulative tables (the image's head)
    slice(L.prob_table, 8, 0, t.prob_table_n);
    const uint64_t pack_ns = ns_since(t0);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "upload");
    cudaEventRecord(ctx->ev_h2d, ctx->stream);

    // One CTA owning all T words of a source writes at most T records.
    uint32_t K = tcfg.direct ? std::max<uint32_t>(ctx->record_slots, tcfg.T) : ctx->record_slots;
    // Multi-CTA circuits (one word per CTA) emit through the record pool.
    uint64_t pool = 0;
    if (!tcfg.direct && !tcfg.split)
        pool = std::max<uint64_t>(ctx->pool_hint,
                                  (2 * t.sources) / gp::kPoolChunk + t.groups * tcfg.emit_warps + 16);
    // Split traversal: walker CTA g owns max_l slabs (one per boundary it may walk).
    const uint64_t slabs = tcfg.split ? t.groups * t.max_l : 0;
    uint64_t ids_cap = std::max<uint64_t>(ctx->ids_hint, 3 * t.sources + 1024);
    DevPlan p{};
    int launches = 0;
    for (int attempt = 0;; attempt++) {
        p = DevPlan{};
        p.img = ctx->d_img;
        p.lay = L;
        p.tot = t;
        p.trav = tcfg;
        p.trav.debug = ctx->trav_debug;
        p.trav_smem = tsmem;
        const size_t need = carve(ctx, p, t, nullptr, K, ids_cap, pool, slabs);
        if ((st = ensure_device(ctx, &ctx->d_ws, &ctx->d_ws_cap, need)) != GP_OK) return st;
        carve(ctx, p, t, ctx->d_ws, K, ids_cap, pool, slabs);
        if (ctx->trav_debug & 4) {  // experiments: per-step walk timestamps of every CTA
            if (!ctx->d_dbg) cudaMalloc(&ctx->d_dbg, (size_t)8192 * 512 * 4 * 8);
            cudaMemsetAsync(ctx->d_dbg, 0, (size_t)8192 * 512 * 4 * 8, ctx->stream);
            p.dbg = t.groups <= 8192 ? ctx->d_dbg : nullptr;
        }
        launches += gp::enqueue_pipeline(p, ctx->stream, &ctx->stage_ev, nullptr, &e);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "kernel launch");
        e = cudaMemcpyAsync(ctx->h_hdr, p.hdr, sizeof(DeviceHeader), cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "device pipeline");
        hdr = *ctx->h_hdr;
        if (attempt > 4) return fail(ctx, GP_ERR_CUDA, "capacity retry loop did not converge");
        if (hdr.pool_overflow) {  // the record pool was too small
            pool = 2 * std::max<uint64_t>(pool, hdr.pool_chunks);
            ctx->pool_hint = pool;
            continue;
        }
        if (hdr.record_overflow) {  // a signature spans more words than inline slots
            K = std::min<uint32_t>(16, std::max<uint32_t>(hdr.record_overflow, 2 * K));
            if (hdr.record_overflow > 16)
                return fail(ctx, GP_ERR_UNSUPPORTED, "signature spans more than 16 detector words");
            ctx->record_slots = K;
            continue;
        }
        if (hdr.num_det_ids == 0xFFFFFFFFu) {  // id capacity overflow
            ids_cap *= 4;
            ctx->ids_hint = ids_cap;
            continue;
        }
        break;
    }
    ctx->last_plan = p;
    ctx->has_plan = true;
    if (p.dbg) {
        const char *path = std::getenv("GP_DEBUG_DUMP");
        std::vector<uint64_t> h((size_t)t.groups * 512 * 4);
        cudaMemcpy(h.data(), p.dbg, h.size() * 8, cudaMemcpyDeviceToHost);
        if (path)
            if (FILE *f = std::fopen(path, "wb")) {
                std::fwrite(h.data(), 8, h.size(), f);
                std::fclose(f);
            }
    }
    const uint64_t E = hdr.num_edges, nd = hdr.num_det_ids, no = hdr.num_obs_ids;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o = (size_t)align16(o + bytes);
        return at;
    };
    const size_t o_det_off = take((E + 1) * 8), o_obs_off = take((E + 1) * 8), o_prob = take(E * 8),
                 o_det = take(nd * 4), o_obs = take(no * 4), o_edge = take((count + 1) * 8);
    if ((st = ensure_host(ctx, &ctx->h_out, &ctx->h_out_cap, o)) != GP_OK) return st;
    auto d2h = [&](size_t off, const void *src, size_t bytes) {
        if (bytes && e == cudaSuccess)
            e = cudaMemcpyAsync(ctx->h_out + off, src, bytes, cudaMemcpyDeviceToHost, ctx->stream);
    };
    d2h(o_det_off, p.o_det_off, (E + 1) * 8);
    d2h(o_obs_off, p.o_obs_off, (E + 1) * 8);
    d2h(o_prob, p.o_prob, E * 8);
    d2h(o_det, p.o_det, nd * 4);
    d2h(o_obs, p.o_obs, no * 4);
    d2h(o_edge, p.o_edge_off, (count + 1) * 8);
    cudaEventRecord(ctx->ev_end, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "download");
    ho.det_off = (uint64_t *)(ctx->h_out + o_det_off);
    ho.obs_off = (uint64_t *)(ctx->h_out + o_obs_off);
    ho.probs = (double *)(ctx->h_out + o_prob);
    ho.det_ids = (uint32_t *)(ctx->h_out + o_det);
    ho.obs_ids = (uint32_t *)(ctx->h_out + o_obs);
    ho.edge_off = (uint64_t *)(ctx->h_out + o_edge);
    if (stats) {
        const double h2d = elapsed_ms(ctx->ev_start, ctx->ev_h2d);
        const double low = elapsed_ms(ctx->ev_h2d, ctx->stage_ev.lowered);
        const double trav = elapsed_ms(ctx->stage_ev.lowered, ctx->stage_ev.traversed);
        const double red = elapsed_ms(ctx->stage_ev.traversed, ctx->stage_ev.reduced);
        const double d2h_ms = elapsed_ms(ctx->stage_ev.reduced, ctx->ev_end);
        *stats = gp_stats{};
        stats->h2d_ns = (uint64_t)(h2d * 1e6);
        stats->lower_ns = pack_ns + (uint64_t)((h2d + low) * 1e6);
        stats->traverse_ns = (uint64_t)(trav * 1e6);
        stats->traverse_kernel_ns = (uint64_t)(trav * 1e6);
        stats->reduce_ns = (uint64_t)((red + d2h_ms) * 1e6);
        stats->kernel_ns = (uint64_t)((low + trav + red) * 1e6);
        stats->d2h_ns = (uint64_t)(d2h_ms * 1e6);
        stats->num_sources = t.sources;
        stats->h2d_bytes = L.total;
        stats->d2h_bytes = sizeof(DeviceHeader) + o;
        stats->kernel_launches = (uint64_t)launches;
        stats->total_ns = ns_since(t0);
    }
    return GP_OK;
}

}  // namespace

extern "C" {

gp_status gp_ctx_create(int device, gp_ctx **out) {
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return GP_ERR_NO_DEVICE;
    }
    if (device < 0 || device >= n) return GP_ERR_NO_DEVICE;
    gp_ctx *ctx = new gp_ctx();
    ctx->device = device;
    cudaSetDevice(device);
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMallocHost(&ctx->h_hdr, sizeof(DeviceHeader)) != cudaSuccess) {
        delete ctx;
        return GP_ERR_CUDA;
    }
    cudaEventCreate(&ctx->ev_start);
    cudaEventCreate(&ctx->ev_h2d);
    cudaEventCreate(&ctx->ev_end);
    cudaEventCreate(&ctx->stage_ev.lowered);
    cudaEventCreate(&ctx->stage_ev.traversed);
    cudaEventCreate(&ctx->stage_ev.reduced);
    *out = ctx;
    return GP_OK;
}

void gp_ctx_destroy(gp_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
    if (ctx->h_out) cudaFreeHost(ctx->h_out);
    if (ctx->h_hdr) cudaFreeHost(ctx->h_hdr);
    if (ctx->d_img) cudaFree(ctx->d_img);
    if (ctx->d_ws) cudaFree(ctx->d_ws);
    if (ctx->d_flush) cudaFree(ctx->d_flush);
    for (cudaEvent_t ev : ctx->prof)
        if (ev) cudaEventDestroy(ev);
    for (cudaEvent_t ev : {ctx->ev_start, ctx->ev_h2d, ctx->ev_end, ctx->stage_ev.lowered, ctx->stage_ev.traversed,
                           ctx->stage_ev.reduced})
        if (ev) cudaEventDestroy(ev);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char *gp_last_error(gp_ctx *ctx) { return ctx ? ctx->err.c_str() : "no context"; }

gp_status gp_ctx_set_option(gp_ctx *ctx, int option, int64_t value) {
    switch (option) {
        case GP_OPT_FORCE_HASH_COLLISIONS:
            ctx->force_collisions = value != 0;
            return GP_OK;
        case GP_OPT_RECORD_SLOTS:
            if (value < 1 || value > 16) return fail(ctx, GP_ERR_INVALID_ARGUMENT, "record slots must be 1..16");
            ctx->record_slots = (uint32_t)value;
            return GP_OK;
        case GP_OPT_SYNC_TIMING:
            return GP_OK;  // stage events are always recorded
        case 99:  // traversal experiments (not part of the ABI contract)
            ctx->trav_debug = (uint32_t)value;
            return GP_OK;
    }
    return fail(ctx, GP_ERR_INVALID_ARGUMENT, "unknown option");
}

gp_status gp_compile(gp_ctx *ctx, const gp_circuit_view *circuit, uint8_t level, gp_dem_view *out,
                     gp_stats *stats) {
    ctx->err.clear();
    HostOut ho{};
    DeviceHeader hdr{};
    gp_status st = run_batch(ctx, circuit, 1, level, ho, hdr, stats);
    if (st != GP_OK) return st;
    out->num_detectors = circuit->num_detectors;
    out->num_observables = circuit->num_observables;
    out->num_edges = hdr.num_edges;
    out->det_offsets = ho.det_off;
    out->det_ids = ho.det_ids;
    out->obs_offsets = ho.obs_off;
    out->obs_ids = ho.obs_ids;
    out->probs = ho.probs;
    return GP_OK;
}

gp_status gp_compile_batch(gp_ctx *ctx, const gp_circuit_view *circuits, size_t count, uint8_t level,
                           gp_dem_batch_view *out, gp_stats *stats) {
    ctx->err.clear();
    HostOut ho{};
    DeviceHeader hdr{};
    gp_status st = run_batch(ctx, circuits, count, level, ho, hdr, stats);
    if (st != GP_OK) return st;
    ctx->out_ndet.resize(count);
    ctx->out_nobs.resize(count);
    for (size_t c = 0; c < count; c++) {
        ctx->out_ndet[c] = circuits[c].num_detectors;
        ctx->out_nobs[c] = circuits[c].num_observables;
    }
    out->num_circuits = count;
    out->edge_offsets = ho.edge_off;
    out->num_detectors = ctx->out_ndet.data();
    out->num_observables = ctx->out_nobs.data();
    out->num_edges = hdr.num_edges;
    out->det_offsets = ho.det_off;
    out->det_ids = ho.det_ids;
    out->obs_offsets = ho.obs_off;
    out->obs_ids = ho.obs_ids;
    out->probs = ho.probs;
    return GP_OK;
}

gp_status gp_replay(gp_ctx *ctx, uint32_t iterations, int flush_l2, gp_stats *stats) {
    if (!ctx->has_plan) return fail(ctx, GP_ERR_INVALID_ARGUMENT, "gp_replay needs a previous successful compile");
    cudaSetDevice(ctx->device);
    constexpr size_t kFlush = 256ull << 20;  // > 126 MB L2
    if (flush_l2 && !ctx->d_flush && cudaMalloc(&ctx->d_flush, kFlush) != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, GP_ERR_OUT_OF_MEMORY, "flush buffer");
    }
    for (cudaEvent_t &ev : ctx->prof)
        if (!ev) cudaEventCreate(&ev);
    std::fill(std::begin(ctx->prof_ns), std::end(ctx->prof_ns), 0);
    uint64_t total = 0, trav = 0;
    int launches = 0;
    for (uint32_t it = 0; it < iterations; it++) {
        if (flush_l2) cudaMemsetAsync(ctx->d_flush, it & 0xFF, kFlush, ctx->stream);
        cudaError_t e;
        launches = gp::enqueue_pipeline(ctx->last_plan, ctx->stream, nullptr, ctx->prof, &e);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "replay");
        for (int k = 1; k < gp::kProfCount; k++)
            ctx->prof_ns[k] += (uint64_t)(elapsed_ms(ctx->prof[k - 1], ctx->prof[k]) * 1e6);
        total += (uint64_t)(elapsed_ms(ctx->prof[0], ctx->prof[gp::kProfCount - 1]) * 1e6);
        trav += (uint64_t)(elapsed_ms(ctx->prof[gp::kProfLower], ctx->prof[gp::kProfEmit]) * 1e6);
    }
    if (stats) {
        *stats = gp_stats{};
        stats->kernel_ns = total;
        stats->traverse_kernel_ns = trav;
        stats->traverse_ns = trav;
        stats->kernel_launches = (uint64_t)launches;
        stats->num_sources = ctx->last_plan.tot.sources;
    }
    return GP_OK;
}

int gp_profile_stages(gp_ctx *ctx, uint64_t *ns, const char **names, int cap) {
    int n = 0;
    for (int k = 1; k < gp::kProfCount && n < cap; k++, n++) {
        if (ns) ns[n] = ctx->prof_ns[k];
        if (names) names[n] = gp::kProfNames[k];
    }
    return n;
}

gp_status gp_circuit_metrics(const gp_circuit_view *v, uint8_t level, gp_metrics *out) {
    *out = gp_metrics{};
    const uint32_t n = v->num_qubits, l = v->num_layers;
    out->base_nodes = (uint64_t)l * 2 * n;
    out->words = ((uint64_t)v->num_detectors + v->num_observables + 63) / 64;
    out->measurements = v->num_measurements;
    std::vector<uint8_t> refs(n);
    for (uint32_t i = 1; i < l; i++) {  // layer i shapes boundary i - 1
        std::fill(refs.begin(), refs.end(), 2);  // idle: X -> X, Z -> Z
        for (uint32_t g = v->gate_offsets[i]; g < v->gate_offsets[i + 1]; g++) {
            const uint32_t q = v->gate_q0[g];
            switch (v->gate_kind[g]) {
                case GP_GATE_CX:
                    refs[q] = 3;
                    refs[v->gate_q1[g]] = 3;
                    break;
                case GP_GATE_R:
                    refs[q] = 0;
                    break;
                case GP_GATE_MR:
                    refs[q] = 1;
                    break;
                default:  // H: 2, M: leaf + X
                    refs[q] = 2;
            }
        }
        for (uint32_t q = 0; q < n; q++) out->succ_refs += refs[q];
    }
    static const uint8_t kDep2[15] = {4, 8, 1, 5, 2, 10, 12, 9, 3, 6, 13, 7, 15, 11, 14};
    for (uint32_t o = 0; o < v->noise_offsets[l]; o++) {
        const uint8_t k = v->noise_kind[o];
        const uint32_t nc = components(k, level);
        out->sources += nc;
        if (k <= GP_NOISE_Z_ERROR) out->source_rows += 1;
        else if (k == GP_NOISE_DEPOLARIZE1) out->source_rows += nc == 2 ? 2 : 4;
        else
            for (uint32_t c = 0; c < nc; c++) out->source_rows += (uint64_t)__builtin_popcount(kDep2[c]);
    }
    for (uint32_t g = 0; g < v->gate_offsets[l]; g++)
        if ((v->gate_kind[g] == GP_GATE_M || v->gate_kind[g] == GP_GATE_MR) && v->gate_flip[g] > 0) {
            out->sources++;
            out->source_rows++;
        }
    return GP_OK;
}

char *gp_serialize_dem(const gp_dem_view *d, size_t *len) {
    // serialize_dem (dem.cpp:144-157) with format_double = std::to_chars
    // shortest round-trip (util.hpp:24-28).
    std::string s;
    s.reserve(d->num_edges * 40 + 1);
    char buf[64];
    for (uint64_t e = 0; e < d->num_edges; e++) {
        s += "error(";
        auto r = std::to_chars(buf, buf + sizeof buf, d->probs[e]);
        s.append(buf, r.ptr);
        s += ')';
        for (uint64_t k = d->det_offsets[e]; k < d->det_offsets[e + 1]; k++) {
            s += " D";
            r = std::to_chars(buf, buf + sizeof buf, d->det_ids[k]);
            s.append(buf, r.ptr);
        }
        for (uint64_t k = d->obs_offsets[e]; k < d->obs_offsets[e + 1]; k++) {
            s += " L";
            r = std::to_chars(buf, buf + sizeof buf, d->obs_ids[k]);
            s.append(buf, r.ptr);
        }
        s += '\n';
    }
    char *out = (char *)std::malloc(s.size() + 1);
    std::memcpy(out, s.data(), s.size());
    out[s.size()] = 0;
    if (len) *len = s.size();
    return out;
}

void *gp_host_alloc(size_t bytes) {
    void *p = nullptr;
    if (cudaMallocHost(&p, bytes ? bytes : 1) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

void gp_host_free(void *p) {
    if (p) cudaFreeHost(p);
}

void gp_free(void *p) { std::free(p); }

}  // extern "C"

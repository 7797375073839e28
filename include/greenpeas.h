/* greenpeas.h -- C ABI of the B200-native DEM compiler (libgreenpeas.so).
 *
 * Drop-in boundary for the reference hot path
 *     demc::Dem demc::compile_circuit(const Circuit &c, CorrelationLevel level,
 *                                     uint32_t threads = 1, CompileStats *stats = nullptr)
 * (/root/reference/proj/core/include/demc/compile.hpp:35-36,
 *  implementation core/src/compile.cpp:23-53).
 *
 * Plain C: status codes, plain pointers and sizes, no exceptions and no torch
 * types. Every entry point lists the reference interface it replaces. The C++
 * shim in include/demc/compile.hpp restores the reference signature on top of
 * this ABI (see INTEGRATION.md for the binding a maintainer would add).
 */
#ifndef GREENPEAS_H
#define GREENPEAS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GP_ABI_VERSION 1

/* Status codes. GP_ERR_INVALID_ARGUMENT carries the reference's
 * std::invalid_argument messages verbatim via gp_last_error():
 *   "circuit exceeds 32-bit node index space"             (stepg.cpp:172-174)
 *   "detector references a measurement without a leaf"    (eec.cpp:44-46)
 *   "observable references a measurement without a leaf"  (eec.cpp:52-54) */
typedef enum gp_status {
    GP_OK = 0,
    GP_ERR_INVALID_ARGUMENT = 1,
    GP_ERR_CUDA = 2,
    GP_ERR_OUT_OF_MEMORY = 3,
    GP_ERR_NO_DEVICE = 4,
    GP_ERR_UNSUPPORTED = 5
} gp_status;

/* circuit.hpp:35 GateKind and circuit.hpp:53 NoiseKind, same numbering. */
enum { GP_GATE_H = 0, GP_GATE_CX = 1, GP_GATE_R = 2, GP_GATE_M = 3, GP_GATE_MR = 4 };
enum { GP_NOISE_X_ERROR = 0, GP_NOISE_Z_ERROR = 1, GP_NOISE_DEPOLARIZE1 = 2, GP_NOISE_DEPOLARIZE2 = 3 };
/* stepg.hpp:28 CorrelationLevel. */
enum { GP_LEVEL_L0 = 0, GP_LEVEL_L1 = 1, GP_LEVEL_L2 = 2 };

/* Flat structure-of-arrays view of demc::Circuit (circuit.hpp:33-97).
 * Layer i owns gates [gate_offsets[i], gate_offsets[i+1]) and noise ops
 * [noise_offsets[i], noise_offsets[i+1]). Detector d owns measurement indices
 * det_meas[det_offsets[d] .. det_offsets[d+1]); observables likewise. The
 * circuit must satisfy demc::validate_layers (circuit.cpp:254-326), exactly as
 * the reference compile_circuit assumes. Caller-owned; not
 * retained after the call. Pinned host memory gives the fastest upload. */
typedef struct gp_circuit_view {
    uint32_t num_qubits;
    uint32_t num_layers;
    uint32_t num_measurements;
    uint32_t num_detectors;
    uint32_t num_observables;
    const uint32_t *gate_offsets; /* [num_layers + 1] */
    const uint8_t *gate_kind;     /* GP_GATE_* */
    const uint32_t *gate_q0;      /* control for CX */
    const uint32_t *gate_q1;      /* CX target; ignored otherwise */
    const int32_t *gate_meas;     /* M/MR absolute record index; ignored otherwise */
    const double *gate_flip;      /* M/MR outcome-flip probability */
    const uint32_t *noise_offsets; /* [num_layers + 1] */
    const uint8_t *noise_kind;     /* GP_NOISE_* */
    const double *noise_prob;
    const uint32_t *noise_q0;
    const uint32_t *noise_q1; /* DEPOLARIZE2 only */
    const uint32_t *det_offsets; /* [num_detectors + 1] */
    const uint32_t *det_meas;
    const uint32_t *obs_offsets; /* [num_observables + 1] */
    const uint32_t *obs_meas;
} gp_circuit_view;

/* Flat view of demc::Dem (dem.hpp:38-52): hyperedges in the reference's
 * canonical order (dem.cpp:122-127), ids strictly ascending within an edge.
 * Offsets are 32-bit (a compile or batch holds < 2^32 ids; larger batches
 * fail with GP_ERR_UNSUPPORTED -- split them).
 * Memory is owned by the context (pinned host) and valid until the next
 * compile call on that context. */
typedef struct gp_dem_view {
    uint32_t num_detectors;
    uint32_t num_observables;
    uint64_t num_edges;
    const uint32_t *det_offsets; /* [num_edges + 1] */
    const uint32_t *det_ids;
    const uint32_t *obs_offsets; /* [num_edges + 1] */
    const uint32_t *obs_ids;
    const double *probs; /* [num_edges] */
} gp_dem_view;

/* A batch result: circuit c owns edges [edge_offsets[c], edge_offsets[c+1])
 * of the concatenated flat DEM (offsets into det_offsets/obs_offsets/probs). */
typedef struct gp_dem_batch_view {
    uint64_t num_circuits;
    const uint64_t *edge_offsets;    /* [num_circuits + 1] */
    const uint32_t *num_detectors;   /* [num_circuits] */
    const uint32_t *num_observables; /* [num_circuits] */
    uint64_t num_edges;
    const uint32_t *det_offsets; /* [num_edges + 1], global */
    const uint32_t *det_ids;
    const uint32_t *obs_offsets; /* [num_edges + 1], global */
    const uint32_t *obs_ids;
    const double *probs;
} gp_dem_batch_view;

/* Mirrors demc::CompileStats (compile.hpp:26-31) and adds the device split. */
typedef struct gp_stats {
    uint64_t lower_ns;    /* host packing + device lowering (STEPG build) */
    uint64_t traverse_ns; /* device: Alg. 1 traversal + signature emission */
    uint64_t reduce_ns;   /* device: dedup + fold + canonical order */
    uint64_t total_ns;    /* wall time of the call, entry to DEM available */
    uint64_t h2d_ns;      /* host->device upload, event-timed */
    uint64_t kernel_ns;   /* all kernels, event-timed */
    uint64_t d2h_ns;      /* device->host download, event-timed */
    uint64_t num_sources; /* error sources (expanded fault mechanisms) */
    uint64_t h2d_bytes;
    uint64_t d2h_bytes;
    uint64_t kernel_launches;
    uint64_t traverse_kernel_ns; /* the traversal kernel alone */
} gp_stats;

typedef struct gp_ctx gp_ctx;

/* Creates a context bound to CUDA device `device`: one stream, pinned host
 * arenas, device workspace. Not thread-safe; use one context per host thread
 * (the reference is reentrant, SPEC.md:71,144 -- contexts restore that). */
gp_status gp_ctx_create(int device, gp_ctx **out);
void gp_ctx_destroy(gp_ctx *ctx);
/* Message of the last failing call on this context ("" if none). */
const char *gp_last_error(gp_ctx *ctx);

/* Context options (test hooks and tuning). */
enum {
    GP_OPT_FORCE_HASH_COLLISIONS = 1, /* every signature hashes to one key: the
                                         reference's injectable HashFn test hook
                                         (dem.hpp:59, test_dem.cpp:94-101) */
    GP_OPT_RECORD_SLOTS = 2,          /* inline sparse-signature slots per source */
    GP_OPT_SYNC_TIMING = 3,           /* 1: event-time each stage into gp_stats */
    GP_OPT_PIPELINE = 4               /* batches of >= 1024 circuits: -1 auto (default), 0 off,
                                         1 on -- sub-batches overlap host packing, upload,
                                         device work and download */
};
gp_status gp_ctx_set_option(gp_ctx *ctx, int option, int64_t value);

/* Replaces demc::compile_circuit (compile.cpp:23-53): circuit in host memory
 * -> DEM in ctx-owned pinned host memory. `level` is a GP_LEVEL_*. `stats`
 * may be NULL. */
gp_status gp_compile(gp_ctx *ctx, const gp_circuit_view *circuit, uint8_t level,
                     gp_dem_view *out, gp_stats *stats);

/* Many independent circuits (e.g. adaptive branch circuits, adaptive.cpp:382-391)
 * in one device pass: equivalent to `count` calls of compile_circuit. */
gp_status gp_compile_batch(gp_ctx *ctx, const gp_circuit_view *circuits, size_t count,
                           uint8_t level, gp_dem_batch_view *out, gp_stats *stats);

/* Branch batches generated on the device (the seeds-in /
 * DEM-out mode of the adaptive workload, adaptive.cpp:382-391): circuit c is
 * the BB memory circuit gp_gen_bb(spec..., branch = first_branch + c) --
 * identical gates, noise, detectors and observables -- but it is built
 * straight into device memory from (seed, branch id): the check subsets are
 * drawn on the GPU (mt19937_64 / seed_seq / uniform_real_distribution
 * restated bit for bit, gp_rng.h) and the upload image is written there, so
 * no host circuit, packing or circuit upload exists. The result equals
 * gp_compile_batch over the host-generated circuits. */
typedef struct gp_bb_spec {
    uint32_t l, m;       /* torus; A = x^a0 + y^a1 + y^a2, B = y^b0 + x^b1 + x^b2 */
    uint32_t a[3], b[3];
    uint32_t rounds;
    uint32_t refresh;    /* full rounds: 0, the last, every refresh-th (0: rounds / 2) */
    int32_t noise_model; /* GP_NOISE_MODEL_* */
    uint32_t reserved;
    double p;
    double check_prob;   /* non-full rounds keep each check with this probability */
    uint64_t seed;
} gp_bb_spec;
gp_status gp_compile_bb_branches(gp_ctx *ctx, const gp_bb_spec *spec, uint64_t first_branch, size_t count,
                                 uint8_t level, gp_dem_batch_view *out, gp_stats *stats);

/* Fault-range sharding of ONE circuit: shard k of n owns the
 * error sources placed in layers [l*k/n, l*(k+1)/n) -- noise ops of those
 * layers and the outcome flips of their measurements. gp_compile_shard walks
 * the circuit (Alg. 1) down to the shard's first layer and emits only the
 * shard's sources, as a PARTIAL TABLE: every nonempty signature with its own
 * probability (unfolded, so a merge is bit-exact: dem.cpp:97-106 folds a
 * group's sorted member probabilities). `memory` chooses where the table is
 * returned: GP_MEM_HOST (pinned host memory) or GP_MEM_DEVICE (the context's
 * device memory, ready for an NCCL gather over NVLink).
 * gp_merge_partials reduces the union of the shards' tables (any order; each
 * part's arrays on the host or on the context's device, per part.memory)
 * into the circuit's DEM -- identical to gp_compile of the whole circuit.
 * Views stay valid until the next call on ctx; merge inputs may be views
 * returned by this ctx. See paper_2604_16613_b200/shard.py. */
enum { GP_MEM_HOST = 0, GP_MEM_DEVICE = 1 };
typedef struct gp_partial_view {
    uint32_t num_detectors;
    uint32_t num_observables;
    uint64_t num_sources;         /* nonempty signatures of the shard */
    uint64_t num_records;
    uint32_t memory;              /* GP_MEM_HOST or GP_MEM_DEVICE */
    uint32_t reserved;
    const double *probs;          /* [num_sources] */
    const uint32_t *rec_offsets;  /* [num_sources + 1] into rec_words / rec_bits */
    const uint32_t *rec_words;    /* [num_records] 64-bit id word (ids 64w .. 64w+63) */
    const uint64_t *rec_bits;     /* [num_records] its bits; detector d = bit d, observable o = bit D+o */
} gp_partial_view;
gp_status gp_compile_shard(gp_ctx *ctx, const gp_circuit_view *circuit, uint8_t level, uint32_t shard,
                           uint32_t nshards, uint32_t memory, gp_partial_view *out, gp_stats *stats);
gp_status gp_merge_partials(gp_ctx *ctx, const gp_partial_view *parts, size_t nparts, gp_dem_view *out,
                            gp_stats *stats);

/* Benchmark hooks (not part of the reference API). gp_replay re-runs the
 * device pipeline `iterations` times on the batch uploaded by the last
 * successful compile on this context: inputs already resident in HBM, outputs
 * left in HBM. flush_l2 != 0 overwrites a 256 MiB scratch buffer before each
 * iteration, outside the timed region. stats->kernel_ns receives the summed
 * device time (CUDA events around each pipeline), traverse_kernel_ns the
 * summed traversal-kernel time, kernel_launches the launches per pipeline. */
gp_status gp_replay(gp_ctx *ctx, uint32_t iterations, int flush_l2, gp_stats *stats);
/* Per-stage device time (ns, summed over the last gp_replay) and stage
 * names; returns the number of stages written (<= cap). */
int gp_profile_stages(gp_ctx *ctx, uint64_t *ns, const char **names, int cap);

/* Roofline accounting inputs of one circuit: N = l * 2n base
 * nodes, N_e = non-sentinel successor references among them, C = base/leaf
 * rows over all source expansions, S = sources (reference count), W, M. */
typedef struct gp_metrics {
    uint64_t base_nodes;
    uint64_t succ_refs;
    uint64_t source_rows;
    uint64_t sources;
    uint64_t words;
    uint64_t measurements;
} gp_metrics;
gp_status gp_circuit_metrics(const gp_circuit_view *circuit, uint8_t level, gp_metrics *out);

/* serialize_dem (dem.cpp:144-157): `error(<shortest round-trip>) D.. L..\n`.
 * Returns a malloc'd NUL-terminated string; release with gp_free. */
char *gp_serialize_dem(const gp_dem_view *dem, size_t *len);

/* 64-bit digest of a DEM for bulk parity checks (host, no device work):
 *   h = 0x6a09e667f3bcc909; absorb(D << 32 | O); absorb(E); per edge in order:
 *   absorb(#dets << 32 | #obs), absorb(each detector id), absorb(each
 *   observable id), absorb(probability bits); absorb(h, w) = splitmix64
 *   finaliser of (h + w + 0x9e3779b97f4a7c15).
 * Equal digests <=> identical serialize_dem text (dem.cpp:144-157) up to hash
 * collisions: ids exact, fp64 bits exact. The reference-side restatement over
 * demc::Dem is oracle/ref_capi.cpp dem_digest. gp_dem_batch_digest writes one
 * digest per circuit of a batch view (out[num_circuits]), on host threads. */
uint64_t gp_dem_digest(const gp_dem_view *dem);
void gp_dem_batch_digest(const gp_dem_batch_view *batch, uint64_t *out);

/* Pinned host allocation helpers (for zero-staging circuit uploads). */
void *gp_host_alloc(size_t bytes);
void gp_host_free(void *p);
void gp_free(void *p);

/* ---- synthetic workload generators (host, outside any timed region) ----
 * Owning circuits in the flat layout. Surface/repetition restate the
 * reference generators (codes.cpp:149-333) so their DEMs are comparable;
 * BB / SI1000 / branch generators are new. */
typedef struct gp_circuit gp_circuit;
enum { GP_NOISE_MODEL_PAPER = 0, /* codes.hpp:30-39 NoiseModel{p} */
       GP_NOISE_MODEL_SI1000 = 1,
       GP_NOISE_MODEL_UNIFORM = 2 /* circuit-level depolarising p */ };
gp_circuit *gp_gen_repetition(uint32_t d, uint32_t rounds, double p);
gp_circuit *gp_gen_surface(uint32_t d, uint32_t rounds, double p, int noise_model, int only_z);
/* Bivariate bicycle code: A = x^a0 + y^a1 + y^a2, B = y^b0 + x^b1 + x^b2 on an
 * l x m torus (gross code [[144,12,12]]: l=12, m=6, a=(3,1,2), b=(3,1,2)).
 * Z-memory, `rounds` syndrome rounds; check_prob < 1 skips each check of a
 * non-full round with probability 1 - check_prob using mt19937_64(seed_seq{
 * seed, seed>>32, branch, branch>>32}) (branch circuits). */
gp_circuit *gp_gen_bb(uint32_t l, uint32_t m, const uint32_t a[3], const uint32_t b[3],
                      uint32_t rounds, double p, int noise_model, double check_prob,
                      uint32_t refresh, uint64_t seed, uint64_t branch);
void gp_circuit_free(gp_circuit *c);
gp_circuit_view gp_circuit_get_view(const gp_circuit *c);
/* Circuit text in the reference grammar (circuit.cpp:328-388 layout). */
char *gp_circuit_serialize(const gp_circuit *c, size_t *len);
/* parse_circuit + validate_layers (circuit.cpp:107-326), natively and on the
 * host pool for large texts: text[len] -> owning circuit (release with
 * gp_circuit_free). On malformed text returns NULL and *error (malloc'd,
 * release with gp_free) holds the reference's message: "line N: ..."
 * (ParseError) or "layer L: ..." (validate_layers' invalid_argument). */
gp_circuit *gp_parse_circuit(const char *text, size_t len, char **error);
/* Annotations of a circuit in declaration order, with their layers (the
 * layout serialize_circuit and demc::Layer::annotations need); valid while
 * the circuit lives. */
typedef struct gp_annotation_view {
    uint32_t layer;
    uint32_t is_observable;
    uint32_t id;
    uint32_t num_meas;
    const uint32_t *meas; /* absolute, ascending */
} gp_annotation_view;
const gp_annotation_view *gp_circuit_annotations(const gp_circuit *c, size_t *count);

#ifdef __cplusplus
}
#endif
#endif

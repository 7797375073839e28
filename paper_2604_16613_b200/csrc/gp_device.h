// gp_device.h -- host-side view of the device pipeline (gp_kernels.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gp_layout.h"

namespace gp {

constexpr uint32_t kPoolChunk = 1024;  // records per pool chunk
constexpr uint32_t kPoolInvalid = 0xFFFFFFFFu;
constexpr uint32_t kHugeCtas = 148;  // CTAs sorting buckets too large for a warp

// Traversal launch configuration (chosen by plan_traversal for a batch).
struct TravCfg {
    uint32_t T;          // 64-bit detector words per CTA (column group width)
    uint32_t R;          // state ring depth (boundaries in flight between warp roles)
    uint32_t NST;        // staging ring depth (boundaries prefetched by the producer)
    uint32_t node_warps, emit_warps;
    uint32_t max_n, max_layer_noise, max_layer_meas, max_l;
    uint32_t direct;     // every circuit fits one group: atomic-free emission
    uint32_t split;      // walk_kernel + emit_kernel (one word per CTA) instead of traverse_kernel
    uint32_t walk_threads, walk_npt;  // walk CTA size; base nodes per node thread (0: generic)
    uint32_t G;          // boundaries per staged group (walk_kernel)
    uint32_t max_comp;   // sources per noise op at this level (6 / 10 / 15): the layer source map
    uint32_t fuse_key;   // direct traversal builds the reduce's sort items (red::key_kernel / scatter_kernel skipped)
    uint32_t wide;       // split traversal with the walk state in global memory (circuits too wide for on-chip state)
    uint32_t debug;      // experiments only: bit0 skip emission work, bit1 skip node work
};

// Every device array used by one compile. Carved from one workspace
// allocation by the host (gp_api.cpp); sizes follow BatchTotals.
struct DevPlan {
    // Uploaded staging image (read-only inputs).
    const uint8_t *img;
    StageLayout lay;
    BatchTotals tot;
    TravCfg trav;
    size_t trav_smem;

    // STEPG IR built on device.
    uint32_t *ell;   // [tot.ell] base-slot ELLPACK (node words, gp_layout.h)
    uint64_t *leaf;  // [tot.leaf] leaf rows, tile-major per circuit (Eq. 3)

    // Noise words as the traversal reads them (8 bytes per op): the image's
    // own array, or -- narrow uploads -- widened into the workspace by lower_kernel.
    uint64_t *noise_w;  // [N] narrow batches only
    __host__ __device__ const uint64_t *noise_words() const {
        return tot.narrow ? noise_w : reinterpret_cast<const uint64_t *>(img + lay.noise);
    }

    // Per source.
    double *prob;      // [S]
    uint32_t *nsrc;    // [N] local source offset of each noise op's first component
    uint32_t *cnt;     // [S] sparse signature words emitted
    uint64_t *rbits;   // [S * K]
    uint32_t *rtile;   // [S * K]
    uint32_t K;        // inline record slots per source
    // Record pool (multi-CTA circuits): the traversal appends (source, word,
    // bits) records in per-warp chunks; slot_kernel files them per source.
    uint4 *pool;          // [pool_chunks_cap * kPoolChunk] {src, word, bits lo, bits hi}
    uint32_t pool_chunks_cap;
    // Split traversal: walker CTA g owns slabs [g * slab_stride, (g + 1) *
    // slab_stride), one per walked boundary (2n u64 words), each with a
    // header {circuit, word, boundary, state}.
    uint64_t *slab;
    uint4 *slab_hdr;
    uint32_t slab_stride, slab_words;
    // Reduce (gp_reduce.cuh), per source: bucket, slot in the bucket, id counts.
    uint32_t *s_bkt, *s_pos;
    int force_collisions;  // test hook: every sort key equal (exact compare decides)
    // Per bucket (circuit, first detector): sources, slot offsets (scan),
    // groups (edges) and their id counts, output offsets (scan).
    uint32_t *bcount;  // [NB + 1]
    uint4 *boff;       // [NB + 1]
    struct alignas(16) ItemStub { uint64_t w[4]; };  // red::Item (32 bytes), sources in bucket order
    ItemStub *items;   // [items_cap]
    uint64_t items_cap;
    uint32_t *ecount;  // [NB]
    uint2 *eids;       // [NB]
    uint4 *oscan;      // [NB + 1]
    // Per group (edge), at the bucket's slots: representative item, probability, id counts.
    uint32_t *e_ndno;
    uint32_t *e_item;  // representative's sort item (its key, or its source's records when incomplete)
    double *e_prob;
    uint32_t *huge;    // [NB] buckets too large for a warp
    // Fused items (trav.fuse_key, full mode): the direct traversal writes each
    // nonempty source's sort item into its circuit's region of `items` (from
    // src_base, in emission order) with its circuit-local bucket in `ibkt`,
    // then lists every bucket's items in `iidx` (boff[b] = {first, count});
    // huge_kernel gathers a listed bucket into `items2` (same positions) and
    // marks its e_item entries with kItem2.
    // Tiny circuits (one CTA does everything, gp_tiny.cuh): enabled by the
    // host for single circuits with D + O <= 64; items capacity (power of 2).
    uint32_t tiny, tiny_cap;
    size_t tiny_smem;
    CircuitMeta tiny_meta;
    uint32_t fused;
    uint32_t fused_move;  // the CTA moves the items into bucket order in items2 (no index list)
    ItemStub *items2;  // [S + 16]
    uint16_t *ibkt;    // [S]
    uint32_t *iidx;    // [S]
    double *ptab3;     // [P * 4] noise probability table: p, p / 3, p / 15 (IEEE division)
    uint64_t ids_cap;

    // Scan scratch.
    uint4 *bsum;       // [S / 2048 + 2]
    uint64_t bsum_cap;

    // Outputs (device; the "output region"), copied to pinned host memory
    // after the header.
    // Offsets are global: this compile's edges / ids / circuits start at
    // base_in[0..3] of the whole batch (a pipelined batch is compiled in
    // sub-batches); write_kernel publishes base_out = base_in + totals.
    uint32_t *o_det_off, *o_obs_off;  // [E_cap + 1] (values global, < 2^32)
    uint32_t *o_det, *o_obs;          // [ids_cap] (local positions)
    double *o_prob;                   // [E_cap]
    uint64_t *o_edge_off;             // [C + 1] (values global)
    uint64_t e_cap;                   // output edge capacity
    const uint64_t *base_in;          // [4] edges, detector ids, observable ids, circuits before this compile
    uint64_t *base_out;               // [4] the same after it
    DeviceHeader *hdr_out;            // final header copy (output region, or mapped host memory)
    // Mapped output (small compiles): copy_out_kernel moves the output region
    // and the header straight into mapped pinned host memory, so the host
    // waits once and reads everything there (no header round trip).
    struct {
        uint32_t *det_off, *obs_off;
        uint64_t *edge_off;
        double *probs;
        uint32_t *det_ids, *obs_ids;
        DeviceHeader *hdr;
    } hmap;
    uint32_t out_mapped;
    // Pipeline mode: kModeFull (circuit -> DEM), kModeShard (sources of
    // layers [shard_lo, shard_hi) -> compact partial table, no reduce),
    // kModeMerge (uploaded partial tables -> DEM: the reduce only).
    uint32_t mode = 0, shard_lo = 0, shard_hi = 0xFFFFFFFFu;  // defaults: the whole circuit
    double *p_prob;      // partial table (kModeShard): [S]
    uint32_t *p_roff;    // [S + 1]
    uint32_t *p_word;    // [S * K]
    uint64_t *p_bits;    // [S * K]
    uint4 *p_scan;       // [S + 1] (nonempty, records) exclusive scan
    // kModeMerge input: the parts' tables concatenated (p_prob [S], p_roff
    // [S + parts], p_word / p_bits [R]); part k = (first source, first
    // offset, first record, records) in m_desc[k].
    const uint4 *m_desc;
    uint32_t m_parts;
    DeviceHeader *hdr;
    uint64_t *dbg;  // experiments only (TravCfg.debug bit 2): per-step walk timestamps
};

enum PipeMode : uint32_t { kModeFull = 0, kModeShard = 1, kModeMerge = 2 };

// Device branch generation (gp_bbgen.cuh): kernel parameters.
struct BBGenParams {
    const uint32_t *xdata, *zdata, *zfinal, *obs_off, *obs_q;  // template (gp_gen.h BBTemplate), device copies
    uint32_t lm, nd, n, rounds, refresh, O, MW, level, C;
    double check_prob, pm;
    uint64_t seed, first;
    uint32_t pi[5];   // probability-table index per channel: p1, p2, pr, pidle, pidle (M/MR/R layers); ~0: off
    uint64_t *masks;  // [C][rounds][2][MW] executed X / Z checks
    uint32_t *counts; // [C][rounds] ne | nz << 16
    uint8_t *img;     // staging image on the device (its head already uploaded)
    StageLayout L;
    uint64_t gates, noise;  // planned batch totals (the last circuit's check)
    uint32_t *err;          // circuits whose fill disagreed with the host plan
};
// Dynamic shared memory of the one-CTA tiny compile (0: does not fit).
size_t tiny_smem_bytes(const BatchTotals &t, const CircuitMeta &m, uint32_t cap);
void launch_bbgen_draw(const BBGenParams &g, cudaStream_t st);
void launch_bbgen_fill(const BBGenParams &g, cudaStream_t st);

struct StageEvents {
    cudaEvent_t lowered, traversed, reduced;
};

// Per-stage profile points (event recorded after each stage) for live
// per-kernel timing inside bench.py; stage names in kProfNames.
enum ProfStage {
    kProfStart = 0,
    kProfMemset,
    kProfLower,
    kProfTraverse,
    kProfEmit,
    kProfKey,
    kProfScanBucket,
    kProfScatter,
    kProfBucket,
    kProfScanOut,
    kProfWrite,
    kProfCount
};
constexpr const char *kProfNames[kProfCount] = {"start",  "memset",      "lower",   "traverse", "emit",    "key",
                                                "scan_bucket", "scatter", "bucket",   "scan_out", "write"};

// Enqueues the whole device pipeline on `stream`: lowering, traversal,
// reduce, canonical order, output gather. Returns the number of kernel
// launches (memsets included). `events` may be null.
// wait_write / written (optional): the write stage waits for / then marks an
// event -- sub-batches on concurrent streams publish their global output
// bases (base_in -> base_out) in order.
int enqueue_pipeline(const DevPlan &p, cudaStream_t stream, const StageEvents *events,
                     const cudaEvent_t *prof, cudaError_t *err, cudaEvent_t wait_write = nullptr,
                     cudaEvent_t written = nullptr);

// Chooses the traversal configuration for a batch (group width, ring depths,
// warp roles) and its dynamic shared memory; false if a circuit is too wide
// for on-chip state (R x T x 2n words).
bool plan_traversal(const BatchTotals &t, int device, TravCfg *cfg, size_t *smem);

}  // namespace gp

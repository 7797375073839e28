// gp_device.h -- host-side view of the device pipeline (gp_kernels.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gp_layout.h"

namespace gp {

constexpr uint32_t kPoolChunk = 1024;  // records per pool chunk
constexpr uint32_t kPoolInvalid = 0xFFFFFFFFu;

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
    uint32_t *rep;     // [S] representative source (group key) or kSuccNone
    uint32_t *gcnt;    // [S] members per representative
    uint2 *ecnt;       // [S] (detector ids, observable ids) per representative
    uint4 *sscan;      // [S] exclusive scan: (edge id, member offset, id offset)

    // Hash table (open addressing, linear probing).
    uint64_t *table;
    uint64_t table_mask;
    int force_collisions;

    // Per edge (capacity S).
    uint32_t *e_src, *e_idoff, *e_nd, *e_no, *e_moff, *e_bucket, *e_circ, *blist, *perm;
    double *e_prob;
    double *mprob;    // [S] member probabilities grouped by edge
    uint4 *pscan;     // [S + 1]
    uint32_t *tid;    // [ids_cap] unsorted-position id lists (bit ids)
    uint64_t ids_cap;

    // Canonical-order buckets.
    uint32_t *bcount;  // [NB]
    uint4 *boff;       // [NB + 1]

    // Scan scratch.
    uint4 *bsum;       // [S / 2048 + 2]
    uint64_t bsum_cap;

    // Outputs (device), copied to pinned host after the header.
    uint64_t *o_det_off, *o_obs_off;  // [S + 1]
    uint32_t *o_det, *o_obs;          // [ids_cap]
    double *o_prob;                   // [S]
    uint64_t *o_edge_off;             // [C + 1]
    DeviceHeader *hdr;
    uint64_t *dbg;  // experiments only (TravCfg.debug bit 2): per-step walk timestamps
};

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
    kProfDedup,
    kProfScanSrc,
    kProfScatter,
    kProfFinalize,
    kProfScanBucket,
    kProfBucketScatter,
    kProfRank,
    kProfScanPos,
    kProfGather,
    kProfCount
};
constexpr const char *kProfNames[kProfCount] = {"start",   "memset",     "lower",          "traverse", "emit", "dedup",
                                                "scan_src", "scatter",   "finalize",       "scan_bucket",
                                                "bucket_scatter", "rank", "scan_pos",      "gather"};

// Enqueues the whole device pipeline on `stream`: lowering, traversal,
// reduce, canonical order, output gather. Returns the number of kernel
// launches (memsets included). `events` may be null.
int enqueue_pipeline(const DevPlan &p, cudaStream_t stream, const StageEvents *events,
                     const cudaEvent_t *prof, cudaError_t *err);

// Chooses the traversal configuration for a batch (group width, ring depths,
// warp roles) and its dynamic shared memory; false if a circuit is too wide
// for on-chip state (R x T x 2n words).
bool plan_traversal(const BatchTotals &t, int device, TravCfg *cfg, size_t *smem);

}  // namespace gp

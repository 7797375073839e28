// gp_device.h -- host-side view of the device pipeline (gp_kernels.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gp_layout.h"

namespace gp {

// Every device array used by one compile. Carved from one workspace
// allocation by the host (gp_api.cpp); sizes follow BatchTotals.
struct DevPlan {
    // Uploaded staging image (read-only inputs).
    const uint8_t *img;
    StageLayout lay;
    BatchTotals tot;

    // STEPG IR built on device.
    uint64_t *ell;   // [tot.ell] base-slot ELLPACK
    uint64_t *leaf;  // [tot.leaf] leaf rows, tile-major per circuit (Eq. 3)

    // Per source.
    double *prob;      // [S]
    uint32_t *cnt;     // [S] sparse signature words emitted
    uint64_t *rbits;   // [S * K]
    uint32_t *rtile;   // [S * K]
    uint32_t K;        // inline record slots per source
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
constexpr const char *kProfNames[kProfCount] = {"start",   "memset",     "lower",          "traverse", "dedup",
                                                "scan_src", "scatter",   "finalize",       "scan_bucket",
                                                "bucket_scatter", "rank", "scan_pos",      "gather"};

// Enqueues the whole device pipeline on `stream`: lowering, traversal,
// reduce, canonical order, output gather. Returns the number of kernel
// launches (memsets included). `events` may be null.
int enqueue_pipeline(const DevPlan &p, cudaStream_t stream, const StageEvents *events,
                     const cudaEvent_t *prof, cudaError_t *err);

// Dynamic shared memory the traversal kernel needs for a batch, and the
// number of staging buffers it will use; returns false if a circuit is too
// wide for on-chip state (2n 64-bit words, double-buffered).
bool traversal_smem(const BatchTotals &t, int device, size_t *bytes, int *stages, int *threads);

}  // namespace gp

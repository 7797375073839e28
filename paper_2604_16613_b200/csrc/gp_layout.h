// gp_layout.h -- device data layout shared by the host packer (gp_api.cpp)
// and the sm_100a kernels (gp_kernels.cu).
//
// A batch of C circuits is uploaded as ONE contiguous staging image (one H2D
// copy) holding the arrays below back to back, each 16-byte aligned and
// padded so that 16-byte-granular bulk copies (cp.async.bulk) may over-read
// by up to 16 bytes. All per-element indices are global across the batch
// unless marked "local".
#pragma once
#include <stdint.h>
#if !defined(__CUDACC__) && !defined(__host__)
#define __host__
#define __device__
#endif

namespace gp {

// Successor encoding of the base-slot STEPG ELLPACK: one u32 per base node.
// Every node of the reference's STEPG has at most two successors through the
// next layer (stepg.cpp:196-234), and one of them, when there are two, is the
// node's own slot at the next boundary (CX: X_c -> {X_c, X_t}, Z_t -> {Z_t,
// Z_c}; M: X -> {leaf, X}). So a node word holds a "self" flag and at most one
// "other" successor -- a base slot at the next boundary or a leaf:
//   bit 31  NOT self (the word 0 is the idle node: X -> X, Z -> Z)
//   bit 30  has other
//   bit 29  other is a leaf (local measurement index) rather than a base slot
//   bits 0-28 the other successor's index
// Only the 2n base slots are materialised: every correlated slot of the
// reference (Y, XZ, ZX, XY, YX, YY, YZ, ZY; stepg.cpp:236-254) is the XOR of
// same-boundary base rows, so sources are expanded onto base rows instead
// (bit-identical; pinned by test_eec.cpp:84-99 and by our oracle parity).
constexpr uint32_t kSuccNotSelf = 1u << 31;
constexpr uint32_t kSuccOther = 1u << 30;
constexpr uint32_t kSuccLeaf = 1u << 29;
constexpr uint32_t kSuccIdx = kSuccLeaf - 1;
constexpr uint32_t kSuccNone = kSuccNotSelf;  // R / Z into M: no successor
constexpr uint32_t kEllIdle = 0;
// ELLPACK rows (one boundary) are padded to a multiple of 4 words so every
// row is a 16-byte-aligned bulk-copy unit.
__host__ __device__ inline uint32_t ell_stride(uint32_t n) { return (2 * n + 3) & ~3u; }

// Gate word: lo = q0 | kind << 29, hi = q1 (CX) or local measurement index.
constexpr uint32_t kGateKindShift = 29;
// Noise word (8 bytes per op): q0 [0,24) | q1 [24,48) | kind [48,50) |
// probability index [50,64) into the batch's probability table (or, in
// wide-probability mode, the op's own fp64 in noise_prob).
constexpr uint32_t kNoiseQubitBits = 24;
constexpr uint64_t kNoiseQubitMask = (1ull << kNoiseQubitBits) - 1;
constexpr uint32_t kNoiseKindShift = 48;
constexpr uint32_t kNoisePidxShift = 50;
constexpr uint32_t kNoisePidxMax = (1u << 14) - 1;  // table entries
__host__ __device__ inline uint32_t noise_q0(uint64_t w) { return (uint32_t)(w & kNoiseQubitMask); }
__host__ __device__ inline uint32_t noise_q1(uint64_t w) { return (uint32_t)(w >> kNoiseQubitBits & kNoiseQubitMask); }
__host__ __device__ inline uint32_t noise_kind(uint64_t w) { return (uint32_t)(w >> kNoiseKindShift & 3); }
__host__ __device__ inline uint32_t noise_pidx(uint64_t w) { return (uint32_t)(w >> kNoisePidxShift); }
// DEPOLARIZE2 component c (0..14) -> mask of (q0 X, q0 Z, q1 X, q1 Z) rows
// (stepg.cpp:66-103 component order), as packed nibbles: no table in memory.
__host__ __device__ inline uint32_t dep2_mask(uint32_t c) { return (uint32_t)(0xEBF7D639CA25184ull >> (4 * c)) & 15u; }

// Narrow upload (BatchTotals.narrow: every circuit of the batch has at most
// 4096 qubits and 32768 measurements, and the batch at most 64 distinct noise
// probabilities): 4-byte op words halve the staging image -- the end-to-end
// path is bound by host memory traffic -- and lower_kernel widens the noise
// words into the workspace for the traversal.
//   gate  : q0 [0,14) | kind [14,17) | hi [17,32) (CX target / local measurement)
//   noise : q0 [0,12) | q1 [12,24) | kind [24,26) | probability index [26,32)
constexpr uint32_t kNarrowMaxQubits = 4096, kNarrowMaxMeas = 32768, kNarrowMaxProbs = 64;
__host__ __device__ inline uint32_t narrow_gate(uint32_t q0, uint32_t kind, uint32_t hi) {
    return q0 | kind << 14 | hi << 17;
}
__host__ __device__ inline uint64_t widen_gate(uint32_t w) {
    return (uint64_t)(w >> 17) << 32 | ((w & 0x3FFFu) | ((w >> 14) & 7u) << kGateKindShift);
}
__host__ __device__ inline uint32_t narrow_noise(uint32_t q0, uint32_t q1, uint32_t kind, uint32_t pidx) {
    return q0 | q1 << 12 | kind << 24 | pidx << 26;
}
__host__ __device__ inline uint64_t widen_noise(uint32_t w) {
    return (uint64_t)(w & 0xFFFu) | (uint64_t)(w >> 12 & 0xFFFu) << kNoiseQubitBits |
           (uint64_t)(w >> 24 & 3u) << kNoiseKindShift | (uint64_t)(w >> 26) << kNoisePidxShift;
}

struct CircuitMeta {
    uint32_t n, l, M, D, O, W;
    uint32_t layer_base;   // index of layer 0 in the layer arrays (l + 1 entries per circuit)
    uint32_t meas_base;    // global index of local measurement 0
    uint32_t det_base;     // index of detector 0 in det_off (D + 1 entries per circuit)
    uint32_t obs_base;     // index of observable 0 in obs_off (O + 1 entries per circuit)
    uint32_t tile_base;    // global tile (64-bit detector column word) index
    uint32_t src_noise;    // noise-derived sources; M flip-source slots follow
    uint32_t bucket_base;  // canonical-order buckets (D + 1 per circuit)
    uint32_t max_layer_noise;  // max noise ops in one layer
    uint64_t src_base;     // global id of source 0
    uint64_t ell_base;     // ELLPACK index of (boundary 0, slot 0); (l - 1) * ell_stride(n) entries
    uint64_t leaf_base;    // leaf matrix index of (tile 0, meas 0); W * M entries, tile-major
    // Host-side packing bases (global element indices of this circuit's slices).
    uint64_t gate_base, noise_base, det_entry_base, obs_entry_base, circ_layer_base;
};

// Leaf rows (one per 64-bit detector word, tile-major) are padded to an even
// length so every row starts 16-byte aligned: a layer's leaf words staged by
// a 16-byte-granular bulk copy then start at local measurement (mb & ~1), and
// the ELLPACK stores leaf successors relative to that start (lower_kernel).
__host__ __device__ inline uint32_t leaf_stride(uint32_t M) { return (M + 1) & ~1u; }

// Offsets (bytes) of every array inside one staging image.
struct StageLayout {
    uint64_t meta;        // CircuitMeta[C]
    uint64_t circ_layer;  // u32[C + 1] cumulative layer count (for warp -> circuit search)
    uint64_t circ_src;    // u64[C + 1] cumulative sources
    uint64_t circ_tile;   // u32[C + 1] cumulative tiles
    uint64_t circ_grp;    // u32[C + 1] cumulative traversal column groups
    uint64_t circ_det;    // u32[C + 1] cumulative detectors
    uint64_t circ_obs;    // u32[C + 1] cumulative observables
    uint64_t circ_bkt;    // u32[C + 1] cumulative reduce buckets (D + 1 per circuit)
    uint64_t lay_gate;    // u32[sum(l + 1)] global gate index of each layer start
    uint64_t lay_noise;   // u32[sum(l + 1)] global noise index
    uint64_t lay_meas;    // u32[sum(l + 1)] local measurement index
    uint64_t gates;       // u64[G] gate words (u32 when narrow)
    uint64_t noise;       // u64[N] noise words (u32 when narrow)
    uint64_t noise_prob;  // f64[N] (wide-probability mode only, else empty)
    uint64_t prob_table;  // f64[P] distinct noise probabilities of the batch
    uint64_t lay_src;     // u32[sum(l + 1)] local source offset of each layer's first op
    uint64_t meas_flip;   // f64[sum M]
    uint64_t det_off;     // u32[sum(D + 1)] global index into det_meas
    uint64_t det_meas;    // u32[] local measurement ids
    uint64_t obs_off;     // u32[sum(O + 1)]
    uint64_t obs_meas;    // u32[]
    uint64_t total;       // bytes
};

struct BatchTotals {
    uint32_t C;
    uint32_t level;
    uint64_t layers;      // sum l
    uint64_t layer_slots; // sum (l + 1)
    uint64_t gates, noise, meas;
    uint64_t det_slots, det_entries, obs_slots, obs_entries;
    uint64_t dets, obss;
    uint64_t tiles;
    uint64_t groups;      // traversal CTAs: sum ceil(W / T)
    uint32_t max_W;
    uint64_t sources;
    uint64_t ell;         // sum (l - 1) * ell_stride(n)
    uint64_t leaf;        // sum W * M
    uint64_t buckets;     // sum (D + 1)
    uint32_t max_n;       // max qubits
    uint32_t max_l;       // max layers
    uint32_t max_layer_noise;
    uint32_t max_layer_meas;
    uint32_t wide_prob;   // 1: per-op fp64 probabilities (table would exceed 14 bits)
    uint32_t prob_table_n;
    uint32_t narrow;      // 1: 4-byte gate / noise words in the image (see narrow_gate)
    uint32_t pad_;
};

// Header written by the device at the end of a compile (read back first).
struct DeviceHeader {
    uint32_t num_edges;
    uint32_t num_det_ids;
    uint32_t num_obs_ids;
    uint32_t num_members;
    uint32_t record_overflow;  // max records seen for one source if > slots, else 0
    uint32_t pool_chunks;      // record-pool chunks handed out by the traversal
    uint32_t pool_overflow;    // chunks requested beyond capacity (re-run larger)
    uint32_t huge_count;       // buckets too large for shared memory
    uint32_t items_overflow;   // nonempty signatures beyond the item capacity (re-run larger)
    uint32_t bad_input;        // merge: malformed partial-table entries (dropped; the call fails)
    uint32_t bucket_next;      // bucket_kernel's work counter (warps take buckets in order)
};

}  // namespace gp

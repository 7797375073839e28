// gp_kernels.cu -- sm_100a device pipeline of the DEM compiler.
//
// Replaces, stage by stage, the body of demc::compile_circuit
// (/root/reference/proj/core/src/compile.cpp:23-53):
//   lower_kernel      lower() (stepg.cpp:165-315) restricted to base slots, plus
//                     EecMatrix::zeroed + init_leaves (eec.cpp:22-58)
//   traverse_kernel   run_backward / Alg. 1 (eec.cpp:64-122) fused with the
//                     per-source signature gather (eec.cpp:130-140), emitting
//                     only nonzero signature words
//   dedup_kernel ..   reduce_packed (dem.cpp:57-142): hash grouping with full
//   gather_kernel     compare, sorted fp64 merge_prob fold, canonical order
// All of it is integer / GF(2) / scalar fp64 work: no tensor cores. Every
// kernel is bound by memory latency or bandwidth; see DESIGN.md.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <mutex>
#include <set>
#include <utility>

#include "gp_device.h"
#include "gp_rng.h"
#include "../../include/greenpeas.h"

namespace gp {

namespace {


// ---------------------------------------------------------------- helpers

__device__ __forceinline__ uint32_t find_u32(const uint32_t *base, uint32_t C, uint32_t x) {
    // largest c in [0, C) with base[c] <= x (base has C + 1 nondecreasing entries)
    uint32_t lo = 0, hi = C;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (base[mid] <= x) lo = mid;
        else hi = mid;
    }
    return lo;
}

// find_u32 by a whole (converged) warp: 32 probes per round, so C = 4,096
// takes 3 rounds of loads instead of 12 dependent ones.
__device__ __forceinline__ uint32_t find_u32_warp(const uint32_t *base, uint32_t C, uint32_t x) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t lo = 0, hi = C;  // base[lo] <= x; the answer is in [lo, hi)
    while (hi - lo > 1) {
        const uint32_t step = (hi - lo + 31) >> 5, pos = lo + lane * step;
        const uint32_t m = __ballot_sync(0xffffffffu, pos < hi && base[pos] <= x);  // lanes 0..k (lane 0: pos = lo)
        lo += (31 - __clz(m)) * step;
        hi = min(hi, lo + step);
    }
    return lo;
}

__device__ __forceinline__ uint32_t find_u64(const uint64_t *base, uint32_t C, uint64_t x) {
    uint32_t lo = 0, hi = C;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (base[mid] <= x) lo = mid;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

// merge_prob (dem.hpp:28-30) with explicit round-to-nearest ops: no FMA
// contraction, bit-identical to the reference's x86-64 (no -march) build.
__device__ __forceinline__ double merge_prob(double a, double b) {
    return __dadd_rn(__dmul_rn(a, __dsub_rn(1.0, b)), __dmul_rn(b, __dsub_rn(1.0, a)));
}

__device__ __forceinline__ uint4 add4(uint4 a, uint4 b) {
    return make_uint4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

// Signature records are slot-major -- slot j of source s at j * S + s -- so
// the first record of consecutive sources is contiguous (most sources have
// one or two records).
__device__ __forceinline__ uint64_t rec_at(const DevPlan &p, uint64_t s, uint32_t j) {
    return (uint64_t)j * p.tot.sources + s;
}

template <class T>
__device__ __forceinline__ const T *arr(const DevPlan &p, uint64_t off) {
    return reinterpret_cast<const T *>(p.img + off);
}

// Components of each noise op (traverse_kernel) as 4-bit masks (bit0 X on
// q0, bit1 Z on q0, bit2 X on q1, bit3 Z on q1); a level keeps a prefix.
// DEPOLARIZE2 (kPairTable, stepg.cpp:49-58): L0 IX IZ XI XX ZI ZZ, L1 adds
// IY XZ YI ZX, L2 adds XY YX YY YZ ZY. DEPOLARIZE1 (stepg.cpp:75-83): X Z, then Y.

__host__ __device__ __forceinline__ uint32_t noise_components(uint32_t kind, uint32_t level) {
    if (kind <= 1) return 1;
    if (kind == 2) return level == 0 ? 2 : 3;
    return level == 0 ? 6 : level == 1 ? 10 : 15;
}

// ---------------------------------------------------------------- PTX wrappers
// Bulk async copy global -> shared, completion counted on an mbarrier
// (the non-tensor TMA path: SASS UBLKCP).

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

constexpr uint32_t kMbarSleepNs = 20000;

// try_wait with a suspend-time hint: the waiting warp sleeps until the phase
// completes (or the hint expires) instead of re-polling, so waiting roles do
// not take issue slots from the working ones.
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t *bar, uint32_t parity, uint32_t ns = kMbarSleepNs) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
        : "memory");
    return ok != 0;
}

// Bounded wait: a protocol bug traps (a CUDA error the host reports) instead
// of hanging the device (a few seconds of suspended try_waits).
// A failed try leaves the warp asleep (__nanosleep, growing to 256 ns):
// measured, the suspend-time hint alone still re-polls often enough to cost
// ~15 % of a traversal's issued instructions.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t spins = 0, ns = 32;
    while (!mbar_try_wait_sleep(bar, parity)) {
        if (++spins > 20000000u) __trap();
        __nanosleep(ns);
        ns = ns < 256 ? 2 * ns : ns;
    }
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    if ((smem_u32(dst) | (uint32_t)(uintptr_t)src | bytes) & 15u) __trap();  // would never complete
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- K1 lowering
// Part A: one warp per (circuit, layer): the gates of layer i fix the base
// successors of boundary i-1 (stepg.cpp:196-234; untouched nodes stay idle =
// word 0 from the memset), M/MR gates publish their flip-source probability,
// noise ops publish their components' probabilities (p, p/3, p/15 with IEEE
// division, stepg.cpp:66-103).
// Part B: one thread per detector / observable toggles its bit into the leaf
// rows of its measurements (init_leaves, eec.cpp:40-58).

// Part A runs a warp per layer (batches: many layers) or, with cta_layer, a
// whole CTA per layer (single circuits: few, wide layers -- the gates split
// over the CTA, the noise ops' component offsets from a CTA scan per chunk).
template <bool cta_layer>
__global__ void lower_kernel(__grid_constant__ const DevPlan p, uint32_t blocks_a) {
    const uint32_t C = p.tot.C;
    const CircuitMeta *meta = arr<CircuitMeta>(p, p.lay.meta);
    if (blockIdx.x < blocks_a) {
        const uint64_t gw = cta_layer ? blockIdx.x : (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
        const uint32_t lane = threadIdx.x & 31;
        // threads of one layer: the warp, or the CTA
        const uint32_t lt = cta_layer ? threadIdx.x : lane, ln = cta_layer ? blockDim.x : 32u;
        if (gw >= p.tot.layers) return;
        const uint32_t *circ_layer = arr<uint32_t>(p, p.lay.circ_layer);
        const uint32_t c = find_u32_warp(circ_layer, C, (uint32_t)gw);  // (gw is warp-uniform)
        const CircuitMeta m = meta[c];
        const uint32_t i = (uint32_t)gw - circ_layer[c];
        const uint32_t li = m.layer_base + i;
        const uint32_t *lay_gate = arr<uint32_t>(p, p.lay.lay_gate);
        const uint32_t *lay_noise = arr<uint32_t>(p, p.lay.lay_noise);
        const uint64_t *gates = arr<uint64_t>(p, p.lay.gates);
        const uint32_t *gates32 = arr<uint32_t>(p, p.lay.gates);
        const bool narrow = p.tot.narrow != 0;
        const double *flip = arr<double>(p, p.lay.meas_flip);
        const uint64_t src_flip = m.src_base + m.src_noise;
        // fused items: the traversal takes each source's probability from the
        // flips / ptab3 itself (no per-source array)
        const bool fused_prob = p.fused && !p.tot.wide_prob;
        if (p.fused && i > 0) {  // batches: this warp owns boundary i - 1's ELL row -- idle (0) first, coalesced
            uint32_t *row = p.ell + m.ell_base + (uint64_t)(i - 1) * ell_stride(m.n);
            for (uint32_t x = lt; x < ell_stride(m.n); x += ln) row[x] = kEllIdle;
            if constexpr (cta_layer) __syncthreads();
            else __syncwarp();
        }
        for (uint32_t g = lay_gate[li] + lt; g < lay_gate[li + 1]; g += ln) {
            const uint64_t w = narrow ? widen_gate(gates32[g]) : gates[g];
            const uint32_t lo = (uint32_t)w, hi = (uint32_t)(w >> 32);
            const uint32_t q = lo & ((1u << kGateKindShift) - 1), kind = lo >> kGateKindShift;
            if ((kind == 3 || kind == 4) && !fused_prob) p.prob[src_flip + hi] = flip[m.meas_base + hi];
            if (i == 0) continue;  // no boundary before layer 0
            uint32_t *e = p.ell + m.ell_base + (uint64_t)(i - 1) * ell_stride(m.n);
            const uint32_t x = 2 * q, z = 2 * q + 1;
            switch (kind) {
                case 0:  // H: X <-> Z
                    e[x] = kSuccNotSelf | kSuccOther | z;
                    e[z] = kSuccNotSelf | kSuccOther | x;
                    break;
                case 1: {  // CX q -> hi: X_c -> {X_c, X_t}, Z_c -> Z_c, X_t -> X_t, Z_t -> {Z_t, Z_c}
                    const uint32_t xt = 2 * hi, zt = 2 * hi + 1;
                    e[x] = kSuccOther | xt;
                    e[z] = kEllIdle;
                    e[xt] = kEllIdle;
                    e[zt] = kSuccOther | z;
                    break;
                }
                case 2:  // R
                    e[x] = kSuccNone;
                    e[z] = kSuccNone;
                    break;
                case 3:  // M: X -> {leaf, X}, Z -> none
                    e[x] = kSuccOther | kSuccLeaf | hi;
                    e[z] = kSuccNone;
                    break;
                default:  // MR: X -> {leaf}, Z -> none
                    e[x] = kSuccNotSelf | kSuccOther | kSuccLeaf | hi;
                    e[z] = kSuccNone;
                    break;
            }
        }
        // Noise ops: component counts -> warp scan -> source offsets (from the
        // layer's base) and per-component probabilities.
        const uint64_t *noise = arr<uint64_t>(p, p.lay.noise);
        const uint32_t *noise32 = arr<uint32_t>(p, p.lay.noise);
        const double *nprob = arr<double>(p, p.lay.noise_prob);
        const double *ptab = arr<double>(p, p.lay.prob_table);
        uint32_t base = arr<uint32_t>(p, p.lay.lay_src)[li];
        for (uint32_t o0 = lay_noise[li]; o0 < lay_noise[li + 1]; o0 += ln) {
            const uint32_t o = o0 + lt;
            const bool act = o < lay_noise[li + 1];
            const uint64_t w = act ? (narrow ? widen_noise(noise32[o]) : noise[o]) : 0;
            if (act && narrow) p.noise_w[o] = w;  // the traversal's 8-byte words
            const uint32_t kind = noise_kind(w);
            const uint32_t k = act ? noise_components(kind, p.tot.level) : 0;
            uint32_t incl = k;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t x = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= (uint32_t)d) incl += x;
            }
            uint32_t chunk = __shfl_sync(0xffffffffu, incl, 31);
            if constexpr (cta_layer) {  // the CTA's chunk: warp totals, then each warp's prefix
                __shared__ uint32_t s_wsum[32];
                const uint32_t wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
                if (lane == 31) s_wsum[wid] = incl;
                __syncthreads();
                uint32_t pre = 0;
                chunk = 0;
                for (uint32_t x = 0; x < nw; x++) {
                    const uint32_t v = s_wsum[x];
                    pre += x < wid ? v : 0u;
                    chunk += v;
                }
                incl += pre;
                __syncthreads();  // (s_wsum is rewritten by the next chunk)
            }
            if (act) {
                const uint32_t off = base + incl - k;
                p.nsrc[o] = off;
                if (!fused_prob) {  // (fused items take them from ptab3 in the traversal)
                    const double pr = p.tot.wide_prob ? nprob[o] : ptab[noise_pidx(w)];
                    const double pe = kind == 2 ? __ddiv_rn(pr, 3.0) : kind == 3 ? __ddiv_rn(pr, 15.0) : pr;
                    double *dst = p.prob + m.src_base + off;
                    for (uint32_t j = 0; j < k; j++) dst[j] = pe;
                }
            }
            base += chunk;
        }
        return;
    }
    // Part B.
    const uint64_t t = (uint64_t)(blockIdx.x - blocks_a) * blockDim.x + threadIdx.x;
    if (t >= p.tot.dets + p.tot.obss) {  // Part C (fused items): component probabilities per table entry
        const uint64_t x = t - p.tot.dets - p.tot.obss;
        if (p.fused && x < p.tot.prob_table_n) {
            const double pr = arr<double>(p, p.lay.prob_table)[x];
            p.ptab3[4 * x] = pr;
            p.ptab3[4 * x + 1] = __ddiv_rn(pr, 3.0);
            p.ptab3[4 * x + 2] = __ddiv_rn(pr, 15.0);
        }
        return;
    }
    if (t < p.tot.dets) {
        const uint32_t c = find_u32(arr<uint32_t>(p, p.lay.circ_det), C, (uint32_t)t);
        const CircuitMeta m = meta[c];
        const uint32_t d = (uint32_t)t - arr<uint32_t>(p, p.lay.circ_det)[c];
        const uint32_t *off = arr<uint32_t>(p, p.lay.det_off) + m.det_base;
        const uint32_t *ms = arr<uint32_t>(p, p.lay.det_meas);
        uint64_t *row = p.leaf + m.leaf_base + (uint64_t)(d >> 6) * leaf_stride(m.M);
        for (uint32_t k = off[d]; k < off[d + 1]; k++)
            atomicXor((unsigned long long *)&row[ms[k]], 1ull << (d & 63));
    } else {
        const uint32_t to = (uint32_t)(t - p.tot.dets);
        const uint32_t c = find_u32(arr<uint32_t>(p, p.lay.circ_obs), C, to);
        const CircuitMeta m = meta[c];
        const uint32_t o = to - arr<uint32_t>(p, p.lay.circ_obs)[c];
        const uint32_t b = m.D + o;
        const uint32_t *off = arr<uint32_t>(p, p.lay.obs_off) + m.obs_base;
        const uint32_t *ms = arr<uint32_t>(p, p.lay.obs_meas);
        uint64_t *row = p.leaf + m.leaf_base + (uint64_t)(b >> 6) * leaf_stride(m.M);
        for (uint32_t k = off[o]; k < off[o + 1]; k++)
            atomicXor((unsigned long long *)&row[ms[k]], 1ull << (b & 63));
    }
}

// ---------------------------------------------------------------- K2 traversal
}  // namespace
#include "gp_reduce.cuh"
#include "gp_traverse.cuh"
#include "gp_walk.cuh"
#include "gp_bbgen.cuh"
#include "gp_tiny.cuh"
namespace {

// Files the traversal's pooled records into per-source slots: the returning
// slot-claim atomics run here, throughput-bound, off the traversal's path.
__global__ void slot_kernel(__grid_constant__ const DevPlan p) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t used = min(p.hdr->pool_chunks, p.pool_chunks_cap);
    if (i >= (uint64_t)used * kPoolChunk) return;
    const uint4 r = p.pool[i];
    if (r.x == kPoolInvalid) return;
    const uint32_t j = atomicAdd(&p.cnt[r.x], 1u);
    if (j < p.K) {
        p.rbits[rec_at(p, r.x, j)] = (uint64_t)r.w << 32 | r.z;
        p.rtile[rec_at(p, r.x, j)] = r.y;
    } else {
        atomicMax(&p.hdr->record_overflow, j + 1);
    }
}

// ---------------------------------------------------------------- scans
// Exclusive scan of uint4 values produced by a functor: reduce tiles ->
// scan tile sums in one CTA -> rescan tiles with offsets.

constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint4 warp_incl_scan(uint4 v) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint4 o;
        o.x = __shfl_up_sync(0xffffffffu, v.x, d);
        o.y = __shfl_up_sync(0xffffffffu, v.y, d);
        o.z = __shfl_up_sync(0xffffffffu, v.z, d);
        o.w = __shfl_up_sync(0xffffffffu, v.w, d);
        if (lane >= (uint32_t)d) v = add4(v, o);
    }
    return v;
}

// Block-wide exclusive scan; returns the exclusive prefix and the block total.
__device__ __forceinline__ uint4 block_excl_scan(uint4 v, uint4 *total) {
    __shared__ uint4 warp_tot[32];
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint4 incl = warp_incl_scan(v);
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        uint4 w = lane < nw ? warp_tot[lane] : make_uint4(0, 0, 0, 0);
        w = warp_incl_scan(w);
        if (lane < nw) warp_tot[lane] = w;
    }
    __syncthreads();
    const uint4 before = wid ? warp_tot[wid - 1] : make_uint4(0, 0, 0, 0);
    *total = warp_tot[nw - 1];
    __syncthreads();
    return add4(before, make_uint4(incl.x - v.x, incl.y - v.y, incl.z - v.z, incl.w - v.w));
}

template <class F>
__global__ void scan_reduce_kernel(F f, uint64_t n, uint4 *bsum) {
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
    uint4 acc = make_uint4(0, 0, 0, 0);
    if (f.active(base)) {
#pragma unroll
        for (int k = 0; k < kScanItems; k++) {
            const uint64_t idx = base + (uint64_t)k * kScanThreads + threadIdx.x;
            if (idx < n) acc = add4(acc, f(idx));
        }
    }
    uint4 tot;
    block_excl_scan(acc, &tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void scan_blocks_kernel(uint4 *bsum, uint32_t nb, uint4 *total_out) {
    const uint32_t per = (nb + blockDim.x - 1) / blockDim.x;
    const uint32_t b0 = threadIdx.x * per, b1 = min(nb, b0 + per);
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (uint32_t b = b0; b < b1; b++) acc = add4(acc, bsum[b]);
    uint4 tot;
    uint4 run = block_excl_scan(acc, &tot);
    for (uint32_t b = b0; b < b1; b++) {
        const uint4 v = bsum[b];
        bsum[b] = run;
        run = add4(run, v);
    }
    if (threadIdx.x == 0) *total_out = tot;
}

template <class F>
__global__ void scan_apply_kernel(F f, uint64_t n, const uint4 *bsum, uint4 *out) {
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
    if (!f.active(base)) return;
    uint4 v[kScanItems];
    uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        const uint64_t idx = base + (uint64_t)threadIdx.x * kScanItems + k;
        v[k] = idx < n ? f(idx) : make_uint4(0, 0, 0, 0);
        acc = add4(acc, v[k]);
    }
    uint4 tot;
    uint4 run = add4(block_excl_scan(acc, &tot), bsum[blockIdx.x]);
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        const uint64_t idx = base + (uint64_t)threadIdx.x * kScanItems + k;
        if (idx < n) out[idx] = run;
        run = add4(run, v[k]);
    }
}

// The whole scan in one launch when it fits one tile (small compiles: a
// launch saved is a few microseconds of latency).
template <class F>
__global__ void scan_single_kernel(F f, uint64_t n, uint4 *out, uint4 *total_out) {
    uint4 v[kScanItems];
    uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        const uint64_t idx = (uint64_t)threadIdx.x * kScanItems + k;
        v[k] = idx < n ? f(idx) : make_uint4(0, 0, 0, 0);
        acc = add4(acc, v[k]);
    }
    uint4 tot;
    uint4 run = block_excl_scan(acc, &tot);
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        const uint64_t idx = (uint64_t)threadIdx.x * kScanItems + k;
        if (idx < n) out[idx] = run;
        run = add4(run, v[k]);
    }
    if (threadIdx.x == 0) *total_out = tot;
}

struct BucketScanF {
    const uint32_t *bcount;
    __device__ bool active(uint64_t) const { return true; }
    __device__ uint4 operator()(uint64_t b) const { return make_uint4(bcount[b], 0, 0, 0); }
};

struct PartialScanF {  // (nonempty sources, records) in source order
    const uint32_t *cnt;
    __device__ bool active(uint64_t) const { return true; }
    __device__ uint4 operator()(uint64_t s) const {
        const uint32_t n = cnt[s];
        return make_uint4(n ? 1u : 0u, n, 0, 0);
    }
};

struct OutScanF {  // (edges, detector ids, observable ids) per bucket, in canonical order
    const uint32_t *ecount;
    const uint2 *eids;
    __device__ bool active(uint64_t) const { return true; }
    __device__ uint4 operator()(uint64_t b) const {
        const uint2 v = eids[b];
        return make_uint4(ecount[b] & 0x7FFFFFFFu, v.x, v.y, 0);  // (bit 31: red::kEdgesInItems)
    }
};

// Zero fills of one compile in one launch (grid-stride over up to 8 ranges).
struct ZeroRanges {
    uint4 *ptr[8];
    uint64_t n16[8];  // 16-byte units
    int count;
};

// Shard mode: the nonempty sources' probabilities and records, compacted in
// source order (the partial table a merge consumes); header = (sources, records).
__global__ void partial_kernel(__grid_constant__ const DevPlan p) {
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t S = p.tot.sources;
    if (s > S) return;
    const uint4 at = p.p_scan[s];
    if (s == S) {  // totals
        p.p_roff[at.x] = at.y;
        p.hdr->num_edges = at.x;
        p.hdr->num_det_ids = at.y;
        return;
    }
    const uint32_t n = p.cnt[s];
    if (n == 0) return;
    if (n > p.K) {
        atomicMax(&p.hdr->record_overflow, n);
        return;
    }
    p.p_prob[at.x] = p.prob[s];
    p.p_roff[at.x] = at.y;
    for (uint32_t j = 0; j < n; j++) {
        p.p_word[at.y + j] = p.rtile[rec_at(p, s, j)];
        p.p_bits[at.y + j] = p.rbits[rec_at(p, s, j)];
    }
}

// Merge mode: the concatenated partial tables -> per-source counts,
// probabilities and slot-major records (the emit stage's layout), one thread
// per source. Malformed entries (no records, more than K, ids outside the
// circuit -- words beyond W or bits beyond D + O in the last word -- or a
// word repeated within an entry) are dropped and counted in hdr->bad_input.
__global__ void unpack_kernel(__grid_constant__ const DevPlan p) {
    const uint64_t S = p.tot.sources;
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) {
        if (s == S) p.cnt[S] = 0;
        return;
    }
    uint32_t lo = 0, hi = p.m_parts;  // part k: m_desc[k].x <= s < m_desc[k + 1].x
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (p.m_desc[mid].x <= s) lo = mid;
        else hi = mid;
    }
    const uint4 d = p.m_desc[lo];
    const uint32_t i = (uint32_t)s - d.x;
    const uint32_t base = p.p_roff[d.y], r0 = p.p_roff[d.y + i] - base, r1 = p.p_roff[d.y + i + 1] - base;
    const uint32_t W = (uint32_t)p.tot.tiles;
    const uint32_t nb = p.tot.dets + p.tot.obss;  // valid bits: ids < D + O
    const uint64_t last_mask = (nb & 63) ? (1ull << (nb & 63)) - 1 : ~0ull;
    bool ok = r1 > r0 && r1 - r0 <= p.K && r1 <= d.w;
    for (uint32_t j = 0; ok && j < r1 - r0; j++) {
        const uint32_t wd = p.p_word[d.z + r0 + j];
        const uint64_t bits = p.p_bits[d.z + r0 + j];
        ok = wd < W && bits != 0 && (wd + 1 < W || (bits & ~last_mask) == 0);
        for (uint32_t i = 0; ok && i < j; i++) ok = p.p_word[d.z + r0 + i] != wd;  // one record per word
    }
    if (!ok) {
        p.cnt[s] = 0;
        atomicAdd(&p.hdr->bad_input, 1u);
        return;
    }
    p.cnt[s] = r1 - r0;
    p.prob[s] = p.p_prob[s];
    for (uint32_t j = 0; j < r1 - r0; j++) {
        p.rtile[rec_at(p, s, j)] = p.p_word[d.z + r0 + j];
        p.rbits[rec_at(p, s, j)] = p.p_bits[d.z + r0 + j];
    }
}

__global__ void zero_kernel(ZeroRanges z) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (int r = 0; r < z.count; r++)
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < z.n16[r]; i += stride)
            z.ptr[r][i] = make_uint4(0, 0, 0, 0);
}

}  // namespace
namespace {

template <class F>
void launch_scan(F f, uint64_t n, uint4 *bsum, uint4 *out, uint4 *total, cudaStream_t st, int *launches) {
    const uint32_t nb = (uint32_t)((n + kScanTile - 1) / kScanTile);
    if (nb == 0) {
        cudaMemsetAsync(total, 0, sizeof(uint4), st);
        return;
    }
    if (nb == 1) {
        scan_single_kernel<<<1, kScanThreads, 0, st>>>(f, n, out, total);
        *launches += 1;
        return;
    }
    scan_reduce_kernel<<<nb, kScanThreads, 0, st>>>(f, n, bsum);
    scan_blocks_kernel<<<1, 1024, 0, st>>>(bsum, nb, total);
    scan_apply_kernel<<<nb, kScanThreads, 0, st>>>(f, n, bsum, out);
    *launches += 3;
}

uint32_t blocks_for(uint64_t n, uint32_t tpb) { return (uint32_t)((n + tpb - 1) / tpb); }

// Opt a kernel into the device's full dynamic shared memory once per
// (function, device), not once per launch (a host call on the latency path).
template <class K>
void smem_optin(K kern) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    if (!done.insert({reinterpret_cast<const void *>(kern), dev}).second) return;
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);  // static shared memory counts against the opt-in limit
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
}

constexpr uint32_t kWalkNpl = 4;  // target nodes per walk thread (issue-bound: more warps)

template <int WPC, class F>
void walk_dispatch_npl(uint32_t npl, F &&launch) {
    switch (npl) {
        case 2: launch(walk::walk_kernel<WPC, 2>); break;
        case 4: launch(walk::walk_kernel<WPC, 4>); break;
        case 8: launch(walk::walk_kernel<WPC, 8>); break;
        case 16: if constexpr (WPC <= 16) { launch(walk::walk_kernel<WPC, 16>); break; } [[fallthrough]];
        default: launch(walk::walk_kernel<WPC, 0>); break;
    }
}

template <class F>
void walk_dispatch(uint32_t wpc, uint32_t npl, F &&launch) {
    switch (wpc) {
        case 1: walk_dispatch_npl<1>(npl, launch); break;
        case 2: walk_dispatch_npl<2>(npl, launch); break;
        case 4: walk_dispatch_npl<4>(npl, launch); break;
        case 8: walk_dispatch_npl<8>(npl, launch); break;
        case 16: walk_dispatch_npl<16>(npl, launch); break;
        default: walk_dispatch_npl<32>(npl, launch); break;
    }
}
constexpr uint32_t kEmitBlocks = 148 * 8;

}  // namespace

bool plan_traversal(const BatchTotals &t, int device, TravCfg *cfg, size_t *smem) {
    int optin = 0, sms = 148;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const size_t budget = (size_t)optin - 2048;  // static shared variables + slack
    TravCfg c{};
    c.max_n = t.max_n;
    c.max_layer_noise = t.max_layer_noise;
    c.max_layer_meas = t.max_layer_meas;
    c.max_l = t.max_l;
    c.max_comp = t.level == 0 ? 6 : t.level == 1 ? 10 : 15;
    const uint32_t n2 = 2 * t.max_n;
    c.node_warps = n2 <= 512 ? 4 : n2 <= 2048 ? 8 : 12;
    c.emit_warps = c.node_warps;
    if (t.C >= 2u * (uint32_t)sms && t.max_W <= 8 && n2 <= 512) {
        // wide-group batches of small circuits: emission (source expansion and
        // the sort items) is the heavier role; 224 threads and a 2-deep state
        // ring fit four CTAs per SM (registers and shared memory), which beats
        // deeper rings (measured: 1 + 5 warps 4.37 ms, 2 + 4 4.41, 1 + 7 with
        // a 3-deep ring 4.48 per 4,096 branches)
        c.node_warps = 1;
        c.emit_warps = 5;
    }
    if (const char *o = std::getenv("GP_TRAV_WARPS")) {  // tuning: "node,emit"
        unsigned a = 0, b = 0;
        if (std::sscanf(o, "%u,%u", &a, &b) == 2 && a && b) {
            c.node_warps = a;
            c.emit_warps = b;
        }
    }
    // Wide groups (one CTA per circuit, atomic-free emission) when the batch
    // alone fills the machine; one word per CTA for single large circuits.
    uint32_t T = 1;
    if (t.C >= 2u * (uint32_t)sms && t.max_W <= 8) T = t.max_W;
    // Batches: shallow rings (more CTAs per SM); single circuits: deep rings
    // (the copy latency of a boundary's stage hides behind NST-1 boundaries).
    static const uint32_t kBatch[][2] = {{2, 3}, {2, 2}, {3, 3}};
    static const uint32_t kSingle[][2] = {{6, 8}, {4, 8}, {4, 6}, {4, 4}, {3, 3}, {2, 2}};
    // split traversal: walk_kernel + emit_kernel; walk_wide_kernel (state in
    // global memory) when even the shallowest on-chip staging does not fit
    auto split = [&]() {
        c.T = 1;
        c.direct = t.max_W <= 1;
        c.split = 1;
        c.wide = 0;
        // Threads per column (a power-of-two number of warps) and unrolled
        // nodes per thread: the fewest warps with <= kWalkNpl nodes each (one
        // warp needs no CTA barrier at all); GP_WALK_WPC overrides (tuning).
        uint32_t wpc = 1;
        while (wpc < 32 && n2 > wpc * 32 * kWalkNpl) wpc *= 2;
        if (const char *o = std::getenv("GP_WALK_WPC")) wpc = std::max(1, std::min(32, std::atoi(o)));
        c.walk_threads = 32 * wpc;
        const uint32_t npl = (n2 + c.walk_threads - 1) / c.walk_threads;
        c.walk_npt = npl <= 2 ? 2 : npl <= 4 ? 4 : npl <= 8 ? 8 : npl <= 16 ? 16 : 0;
        // Deepest staging that fits: groups of G boundaries, NST groups in flight.
        static const uint32_t kOpts[][2] = {{3, 8}, {2, 8}, {3, 4}, {2, 4}, {2, 2}, {2, 1}};
        if (!std::getenv("GP_WALK_WIDE"))  // (tests: force the global-state walk)
            for (const auto &o : kOpts) {
                const walk::WalkDims d(o[0], o[1], t.max_n, t.max_layer_meas, t.max_l);
                if (d.total_bytes() <= budget) {
                    c.NST = o[0];
                    c.G = o[1];
                    c.R = 2;
                    *cfg = c;
                    *smem = d.total_bytes();
                    return true;
                }
            }
        c.wide = 1;
        c.walk_threads = 1024;
        c.NST = c.G = 1;
        c.R = 2;
        *cfg = c;
        *smem = (size_t)((t.max_l + 4) & ~3u) * 5 + 64;  // layer table + liveness flags
        return true;
    };
    if (T == 1) return split();
    for (;; T = (T + 1) / 2) {
        const bool batch = T > 1;
        const uint32_t(*opts)[2] = batch ? kBatch : kSingle;
        const int nopt = batch ? 3 : 6;
        uint32_t force_r = 0, force_n = 0;  // tuning: GP_TRAV_RN="R,NST"
        if (const char *o = std::getenv("GP_TRAV_RN")) std::sscanf(o, "%u,%u", &force_r, &force_n);
        for (int o = 0; o < nopt; o++) {
            uint32_t R = opts[o][0], N = opts[o][1];
            if (force_r && force_n) R = force_r, N = force_n;
            // the layer source -> op map is used only by source-major emission
            // (several words per CTA, every word of the circuit: TM > 1 && direct)
            const uint32_t comp = (T > 1 && t.max_W <= T) ? c.max_comp : 0;
            // a direct CTA owns its circuit's buckets: the key pass is fused
            const bool fuse = T > 1 && t.max_W <= T && t.sources < (1ull << 31) && !std::getenv("GP_NO_FUSED_KEY");
            const trav::Dims d(T, R, N, t.max_n, t.max_layer_meas, t.max_layer_noise, t.max_l, comp, fuse);
            if (d.total_bytes() <= budget) {
                c.max_comp = comp;
                c.fuse_key = fuse;
                c.T = T;
                c.R = R;
                c.NST = N;
                c.direct = t.max_W <= T;
                *cfg = c;
                *smem = d.total_bytes();
                return true;
            }
        }
        if (T == 1) return split();  // (the fused kernel's ring does not fit)
    }
}

int enqueue_pipeline(const DevPlan &p, cudaStream_t st, const StageEvents *ev, const cudaEvent_t *prof,
                     cudaError_t *err, cudaEvent_t wait_write, cudaEvent_t written) {
    int launches = 0;
    auto mark = [&](int k) {
        if (prof) cudaEventRecord(prof[k], st);
    };
    mark(kProfStart);
    if (p.tiny) {  // one CTA: lowering, Alg. 1, emission, reduce, output (gp_tiny.cuh)
        smem_optin(tiny::tiny_kernel);
        static const int tt = std::getenv("GP_TINY_THREADS") ? std::atoi(std::getenv("GP_TINY_THREADS")) : 0;
        const uint32_t threads = tt >= 64 && tt <= (int)tiny::kThreads ? (uint32_t)tt & ~31u : tiny::kThreads;
        tiny::tiny_kernel<<<1, threads, p.tiny_smem, st>>>(p);
        if (prof)
            for (int k = kProfMemset; k < kProfCount; k++) mark(k);
        if (ev) cudaEventRecord(ev->reduced, st);  // (one kernel: no stage split; the host reads `reduced` only)
        *err = cudaGetLastError();
        return 1;
    }
    const uint64_t S = p.tot.sources, NB = p.tot.buckets;
    // Zero fills (one launch): ELLPACK (idle nodes are word 0), leaf rows,
    // per-source record counts, bucket counts, the header.
    {
        ZeroRanges z{};
        auto add = [&](void *ptr, uint64_t bytes) {
            if (!bytes) return;
            z.ptr[z.count] = (uint4 *)ptr;
            z.n16[z.count] = (bytes + 15) / 16;
            z.count++;
        };
        if (p.mode != kModeMerge) {  // (merge: counts and records are uploaded)
            // (batches with fused items: each ELL row is idle-filled by its
            // lowering warp; a single circuit's few layer warps would
            // serialise that, the fill kernel spreads it)
            if (!p.fused) add(p.ell, p.tot.ell * 4);
            add(p.leaf, p.tot.leaf * 8);
            // fused items: records are written (and read) only for incomplete keys
            if (!p.fused) add(p.cnt, S * 4 + 4);
        }
        // fused items: the traversal files every bucket it sees ({first, count}); the rest stay empty
        if (p.fused) add(p.boff, (NB + 1) * 16);
        else add(p.bcount, NB * 4 + 4);
        add(p.hdr, sizeof(DeviceHeader));
        uint64_t units = 0;
        for (int r = 0; r < z.count; r++) units = std::max(units, z.n16[r]);
        zero_kernel<<<(uint32_t)std::min<uint64_t>(blocks_for(units, 256), 148 * 8), 256, 0, st>>>(z);
        launches++;
    }
    mark(kProfMemset);

    if (p.mode == kModeMerge) {  // partial tables in: unpack, then the reduce only
        unpack_kernel<<<(uint32_t)blocks_for(S + 1, 256), 256, 0, st>>>(p);
        launches++;
        goto reduce;
    }
    // K1 lowering.
    {
        const uint32_t tpb = 256;
        // a CTA per layer when a warp per layer would not fill the machine
        const uint32_t cta_layer = p.tot.layers < 148u * 8u ? 1u : 0u;
        const uint32_t ba = cta_layer ? (uint32_t)p.tot.layers : blocks_for(p.tot.layers, tpb / 32);
        const uint32_t bb = blocks_for(p.tot.dets + p.tot.obss + (p.fused ? p.tot.prob_table_n : 0), tpb);
        if (ba + bb) {
            if (cta_layer) lower_kernel<true><<<ba + bb, tpb, 0, st>>>(p, ba);
            else lower_kernel<false><<<ba + bb, tpb, 0, st>>>(p, ba);
            launches++;
        }
    }
    mark(kProfLower);
    if (ev) cudaEventRecord(ev->lowered, st);

    // K2 traversal.
    if (p.tot.groups && p.trav.split) {
        auto launch = [&](auto kern) {
            smem_optin(kern);
            kern<<<(uint32_t)p.tot.groups, p.trav.walk_threads, p.trav_smem, st>>>(p, p.trav);
        };
        if (p.trav.wide) {
            smem_optin(walk::walk_wide_kernel);
            walk::walk_wide_kernel<<<(uint32_t)p.tot.groups, 1024, p.trav_smem, st>>>(p, p.trav);
        } else {
            walk_dispatch(p.trav.walk_threads / 32, p.trav.walk_npt, launch);
        }
        mark(kProfTraverse);
        walk::emit_kernel<<<kEmitBlocks, 256, 0, st>>>(p);
        launches += 2;
    } else if (p.tot.groups) {
        const TravCfg &c = p.trav;
        const int threads = 32 * (1 + (int)c.node_warps + (int)c.emit_warps);
        const uint32_t tm = c.T <= 1 ? 1 : c.T <= 2 ? 2 : c.T <= 4 ? 4 : c.T <= 6 ? 6 : 8;
        auto launch = [&](auto kern) {
            smem_optin(kern);
            kern<<<(uint32_t)p.tot.groups, threads, p.trav_smem, st>>>(p, c);
        };
        if (tm == 1) launch(trav::traverse_kernel<1>);
        else if (tm == 2) launch(trav::traverse_kernel<2>);
        else if (tm == 4) launch(trav::traverse_kernel<4>);
        else if (tm == 6) launch(trav::traverse_kernel<6>);  // (6-word circuits: [[72,12,6]] branches)
        else launch(trav::traverse_kernel<8>);
        launches++;
        if (p.pool_chunks_cap) {
            slot_kernel<<<(uint32_t)((uint64_t)p.pool_chunks_cap * kPoolChunk / 256), 256, 0, st>>>(p);
            launches++;
        }
    }
    if (!p.trav.split) mark(kProfTraverse);
    mark(kProfEmit);
    if (ev) cudaEventRecord(ev->traversed, st);
    if (p.mode == kModeShard) {  // compact partial table of the shard's nonempty sources
        uint4 *ptot = p.bsum + p.bsum_cap - 4;
        launch_scan(PartialScanF{p.cnt}, S + 1, p.bsum, p.p_scan, &ptot[2], st, &launches);
        partial_kernel<<<(uint32_t)std::max<uint64_t>(blocks_for(S + 1, 256), 1), 256, 0, st>>>(p);
        launches++;
        if (ev) cudaEventRecord(ev->reduced, st);
        *err = cudaGetLastError();
        return launches;
    }
reduce:

    // K3 reduce (gp_reduce.cuh): bucket by (circuit, first detector) with a
    // counting sort, sort + group + fold each bucket on chip, write in order.
    const uint32_t tpb = 256;
    uint4 *totals = p.bsum + p.bsum_cap - 4;  // scan totals live at the end of bsum
    const uint32_t sgrid = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(blocks_for(S, tpb), 1), 148 * 32);
    if (!p.fused) {  // (fused items: keys, bucket lists and items come from the traversal)
        red::key_kernel<<<sgrid, tpb, 0, st>>>(p), launches++;
        mark(kProfKey);
        launch_scan(BucketScanF{p.bcount}, NB + 1, p.bsum, p.boff, &totals[0], st, &launches);
        mark(kProfScanBucket);
        // (512-thread CTAs measure best for the scatter, 128 for the write)
        const uint32_t g512 = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(blocks_for(S, 512), 1), 148 * 16);
        red::scatter_kernel<<<g512, 512, 0, st>>>(p), launches++;
    } else {
        mark(kProfKey);
        mark(kProfScanBucket);
    }
    mark(kProfScatter);
    {
        const uint64_t ctas = (NB + red::kBucketThreads / 32 - 1) / (red::kBucketThreads / 32);
        const char *be = std::getenv("GP_BUCKET_CTAS");  // (tuning)
        const uint64_t cap = be ? (uint64_t)std::max(1, std::atoi(be)) : 148 * 16;
        red::bucket_kernel<<<(uint32_t)std::min<uint64_t>(std::max<uint64_t>(ctas, 1), cap), red::kBucketThreads, 0,
                             st>>>(p);
        smem_optin(red::huge_kernel);
        // (listed buckets: over kWarpItems sources, or holding an incomplete key)
        const uint32_t hgrid = (uint32_t)std::min<uint64_t>(kHugeCtas, std::max<uint64_t>(1, S / 64));
        red::huge_kernel<<<hgrid, 256, red::kHugeSmem, st>>>(p);
        launches += 2;
    }
    mark(kProfBucket);
    launch_scan(OutScanF{p.ecount, p.eids}, NB, p.bsum, p.oscan, &totals[1], st, &launches);
    mark(kProfScanOut);
    if (wait_write) cudaStreamWaitEvent(st, wait_write, 0);  // the previous sub-batch's bases
    {
        // buckets per warp: 32 for batches; single circuits keep >= ~4,700
        // warps (32 per SM) busy with fewer
        uint32_t cb = 32;
        while (cb > 1 && NB < (uint64_t)cb * 148 * 32) cb >>= 1;
        const uint64_t threads = std::max<uint64_t>((NB + cb - 1) / cb * 32, p.tot.C + 1);
        red::write_kernel<<<(uint32_t)std::min<uint64_t>(blocks_for(threads, 128), 148 * 256), 128, 0, st>>>(
            p, &totals[1], cb);
        launches++;
    }
    mark(kProfWrite);
    if (written) cudaEventRecord(written, st);
    if (p.out_mapped) {
        const char *ce = std::getenv("GP_COPY_CTAS");  // (tuning)
        const uint32_t cc = ce ? (uint32_t)std::max(1, std::atoi(ce)) : 32u;
        red::copy_out_kernel<<<cc, 256, 0, st>>>(p), launches++;
    }
    if (ev) cudaEventRecord(ev->reduced, st);
    *err = cudaGetLastError();
    return launches;
}

size_t tiny_smem_bytes(const BatchTotals &t, const CircuitMeta &m, uint32_t cap) {
    const tiny::Head h = tiny::head_of(m.l, m.D, m.O, (uint32_t)t.det_entries, (uint32_t)t.obs_entries,
                                       t.prob_table_n, 0, 0, 0, t.wide_prob != 0);
    return tiny::Dims{2 * m.n, m.l, m.M, cap, (uint32_t)h.bytes()}.bytes();
}

void launch_bbgen_draw(const BBGenParams &g, cudaStream_t st) {
    if (g.C) bbgen::bbgen_draw_kernel<<<(g.C + 127) / 128, 128, 0, st>>>(g);
}

void launch_bbgen_fill(const BBGenParams &g, cudaStream_t st) {
    constexpr uint32_t kWarps = 4;  // branches per CTA
    const size_t smem = (size_t)kWarps * bbgen::fill_smem_words(g.n, g.lm) * 4;
    if (smem > 48 * 1024) cudaFuncSetAttribute(bbgen::bbgen_fill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (g.C) bbgen::bbgen_fill_kernel<<<(g.C + kWarps - 1) / kWarps, 32 * kWarps, smem, st>>>(g);
}

}  // namespace gp

// gp_walk.cuh -- K2 split traversal (sm_100a), included by gp_kernels.cu.
//
// Used when a circuit's detector words are spread over many CTAs (single
// large circuits, small batches): one CTA per 64-bit detector word. The fused
// traverse_kernel (gp_traverse.cuh) spends most of each boundary in its emit
// warps there (ncu: node warps spin on the state ring while emit warps expand
// every noise op of the layer), so the two halves of the reference's work are
// split into two kernels that each run at their own speed:
//
//   walk_kernel   Alg. 1 only (run_backward / update_cell, eec.cpp:64-122):
//                 one thread per base node, state double-buffered in shared
//                 memory, the boundary's ELLPACK slice and leaf words staged
//                 NST boundaries ahead by one producer lane with cp.async.bulk.
//                 Each live boundary's column is also written to a global slab
//                 (L2-resident) -- one named barrier per boundary, nothing else.
//   emit_kernel   the per-source signature gather (eec.cpp:130-140;
//                 compile.cpp:34-39) for every noise op placed at a live
//                 boundary, over all SMs: <= 4 base rows per component
//                 (correlated slots are XORs of base rows, stepg.cpp:236-254),
//                 nonzero words filed straight into per-source record slots.
//                 Measurement-flip sources (stepg.cpp:270-272) come from the
//                 leaf rows, one record per (measurement, word).

namespace walk {

__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint64_t lds_u64(uint32_t a) {
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_u64(uint32_t a, uint64_t v) {
    asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}

constexpr uint32_t kSlabLive = 1, kSlabZero = 2, kSlabDead = 0;

// Shared memory: the partner-read state (double-buffered), NST stages of G
// boundaries each (ELLPACK rows, then the leaf words of those layers), the
// stage barriers, the circuit's layer -> measurement table and per-step
// liveness flags.
struct WalkDims {
    uint32_t NST, G, n2, estride, leaf_w, lay_w;
    __host__ __device__ WalkDims(uint32_t nst, uint32_t g, uint32_t max_n, uint32_t max_meas, uint32_t max_l)
        : NST(nst),
          G(g),
          n2(2 * max_n),
          estride(ell_stride(max_n)),
          leaf_w((g * max_meas + 3) & ~1u),
          lay_w((max_l + 4) & ~3u) {}
    __host__ __device__ size_t state_bytes() const { return (size_t)2 * n2 * 8; }
    __host__ __device__ size_t stage_bytes() const { return (size_t)G * estride * 4 + (size_t)leaf_w * 8; }
    __host__ __device__ size_t total_bytes() const {
        return state_bytes() + NST * stage_bytes() + NST * 16 + (size_t)lay_w * 4 + lay_w + 64;
    }
    __device__ uint64_t *state(uint8_t *base, uint32_t r) const {
        return reinterpret_cast<uint64_t *>(base) + (size_t)r * n2;
    }
    __device__ uint8_t *stage(uint8_t *base, uint32_t k) const {
        return base + state_bytes() + (size_t)k * stage_bytes();
    }
    __device__ uint32_t *ell(uint8_t *base, uint32_t k) const { return reinterpret_cast<uint32_t *>(stage(base, k)); }
    __device__ uint64_t *leaf(uint8_t *base, uint32_t k) const {
        return reinterpret_cast<uint64_t *>(stage(base, k) + (size_t)G * estride * 4);
    }
    __device__ uint64_t *bars(uint8_t *base) const {
        return reinterpret_cast<uint64_t *>(base + state_bytes() + NST * stage_bytes());
    }
    __device__ uint32_t *mbal(uint8_t *base) const { return reinterpret_cast<uint32_t *>(bars(base) + NST); }
    __device__ uint32_t *lay(uint8_t *base) const { return reinterpret_cast<uint32_t *>(bars(base) + 2 * NST); }
    __device__ uint8_t *live(uint8_t *base) const { return reinterpret_cast<uint8_t *>(lay(base) + lay_w); }
};

// NPL > 0: thread t owns base nodes t, t + blockDim, ... (NPL of them) and
// keeps their previous-boundary values in registers, so only the "other"
// successor is read from shared memory. NPL == 0: generic loop.
template <int WPC, int NPL>
__global__ void __launch_bounds__(32 * WPC) walk_kernel(__grid_constant__ const DevPlan p, TravCfg cfg) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ CircuitMeta s_meta;
    __shared__ uint32_t s_min_m, s_max_m, s_grp, s_circ;
    __shared__ uint64_t s_zero;  // read by nodes without an "other" successor
    __shared__ volatile uint32_t s_vote[3];

    const WalkDims L(cfg.NST, cfg.G, cfg.max_n, cfg.max_layer_meas, cfg.max_l);
    const uint32_t tid = threadIdx.x;

    if (tid == 0) {
        const uint32_t *circ_grp = arr<uint32_t>(p, p.lay.circ_grp);
        const uint32_t c = find_u32(circ_grp, p.tot.C, blockIdx.x);
        s_meta = arr<CircuitMeta>(p, p.lay.meta)[c];
        s_grp = blockIdx.x - circ_grp[c];
        s_circ = c;
        s_min_m = 0xFFFFFFFFu;
        s_max_m = 0;
        s_zero = 0;
        s_vote[0] = s_vote[1] = s_vote[2] = 0;
    }
    __syncthreads();
    const CircuitMeta m = s_meta;
    const uint32_t word = s_grp, n2 = 2 * m.n, circ_id = s_circ;
    uint4 *hdrs = p.slab_hdr + (uint64_t)blockIdx.x * p.slab_stride;

    {  // measurement window of the word's detectors / observables
        const uint32_t b0 = word * 64, b1 = min(b0 + 64, m.D + m.O);
        const uint32_t *doff = arr<uint32_t>(p, p.lay.det_off) + m.det_base;
        const uint32_t *dms = arr<uint32_t>(p, p.lay.det_meas);
        uint32_t lo = 0xFFFFFFFFu, hi = 0;
        for (uint32_t d = b0 + tid; d < min(b1, m.D); d += blockDim.x)
            for (uint32_t k = doff[d]; k < doff[d + 1]; k++) {
                lo = min(lo, dms[k]);
                hi = max(hi, dms[k]);
            }
        const uint32_t *ooff = arr<uint32_t>(p, p.lay.obs_off) + m.obs_base;
        const uint32_t *oms = arr<uint32_t>(p, p.lay.obs_meas);
        for (uint32_t b = max(b0, m.D); b < b1; b++)
            for (uint32_t k = ooff[b - m.D] + tid; k < ooff[b - m.D + 1]; k += blockDim.x) {
                lo = min(lo, oms[k]);
                hi = max(hi, oms[k]);
            }
        if (lo != 0xFFFFFFFFu) {
            atomicMin(&s_min_m, lo);
            atomicMax(&s_max_m, hi);
        }
    }
    __syncthreads();
    const uint32_t min_m = s_min_m, max_m = s_max_m;
    if (min_m == 0xFFFFFFFFu) {  // every column of the word is zero: no slabs
        for (uint32_t x = tid; x < p.slab_stride; x += blockDim.x) hdrs[x] = make_uint4(0, 0, 0, kSlabDead);
        return;
    }

    uint32_t *lay_meas = L.lay(smem);
    {
        const uint32_t *gm = arr<uint32_t>(p, p.lay.lay_meas) + m.layer_base;
        for (uint32_t i = tid; i <= m.l; i += blockDim.x) lay_meas[i] = gm[i];
    }
    __syncthreads();
    auto layer_of = [&](uint32_t mm) {
        uint32_t lo = 0, hi = m.l;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (lay_meas[mid] <= mm) lo = mid;
            else hi = mid;
        }
        return (int)lo;
    };
    const int first_layer = layer_of(min_m);
    const int b_hi = layer_of(max_m) - 1;
    const int G = (int)L.G;
    // Fault-range shard [shard_lo, shard_hi): boundaries below shard_lo are
    // never walked, words whose leaves all lie below it not at all.
    const int b_lo = (int)min(p.shard_lo, 0x7FFFFFFFu);
    const int ngroups = b_hi >= b_lo ? (b_hi + G) / G : 0;

    uint64_t *full = L.bars(smem);
    uint32_t *mbal = L.mbal(smem);
    uint8_t *s_live = L.live(smem);
    if (tid == 0) {
        for (uint32_t k = 0; k < L.NST; k++) mbar_init(&full[k], 1);
        mbar_fence_init();
    }
    {  // state slot 1 plays S_{b_hi+1} = 0 for the first boundary
        uint64_t *z = L.state(smem, 1);
        for (uint32_t x = tid; x < n2; x += blockDim.x) z[x] = 0;
    }
    __syncthreads();

    const uint32_t estride = ell_stride(m.n);
    const uint32_t *ell = p.ell + m.ell_base;
    const uint64_t *leaf = p.leaf + m.leaf_base + (uint64_t)word * leaf_stride(m.M);  // 16-byte aligned row
    // Producer (thread 0): stage group q -- boundaries [lo, top], top = b_hi -
    // q*G -- as one contiguous ELLPACK block plus the leaf words of layers
    // lo+1 .. top+1 from their aligned start.
    auto issue = [&](int q, uint32_t k) {
        const int top = b_hi - q * G, lo = max(0, top - G + 1);
        const uint32_t mb = lay_meas[lo + 1] & ~1u, me = lay_meas[top + 2];
        const uint32_t lb = me > mb ? ((me - mb + 1) & ~1u) * 8 : 0;
        const uint32_t eb = (uint32_t)(top - lo + 1) * estride * 4;
        mbal[k] = mb;
        fence_proxy_async();
        mbar_arrive_expect_tx(&full[k], eb + lb);
        bulk_g2s(L.ell(smem, k), ell + (uint64_t)lo * estride, eb, &full[k]);
        if (lb) bulk_g2s(L.leaf(smem, k), leaf + mb, lb, &full[k]);
    };
    const bool producer = tid == 0;
    int issued = 0;
    if (producer)
        for (; issued < (int)L.NST && issued < ngroups; issued++) issue(issued, (uint32_t)issued);

    // Lockstep over boundaries. A column is walked by WPC = blockDim/32 warps:
    // with one warp the per-boundary sync is __syncwarp and the zero test a
    // vote; with more, one named barrier and per-warp vote flags (three
    // rotating slots: a slot is cleared two boundaries after it was read).
    // One stage wait per group of G boundaries; thread 0 refills the stage a
    // group released.
    const uint32_t nthreads = blockDim.x;  // == 32 * WPC
    constexpr bool one_warp = WPC == 1;
    uint64_t own[NPL > 0 ? NPL : 1];
#pragma unroll
    for (int i = 0; i < (NPL > 0 ? NPL : 1); i++) own[i] = 0;
    uint64_t *slab0 = p.slab + (uint64_t)blockIdx.x * p.slab_stride * p.slab_words;
    const uint32_t st0 = smem_u32(L.state(smem, 0)), zero0 = smem_u32(&s_zero);
    uint32_t k = 0, par = 0;
    int j = 0, consumed = ngroups;
    uint32_t vslot = 0;  // j % 3
    bool stopped = false;
    uint64_t *dbg = (p.dbg && tid == 0) ? p.dbg + (uint64_t)blockIdx.x * 512 * 4 : nullptr;
    for (int q = 0; q < ngroups && !stopped; q++) {
        const int top = b_hi - q * G, lo = max(0, top - G + 1);
        if (dbg && j < 512) dbg[j * 4 + 0] = clock64();
        mbar_wait(&full[k], par);
        if (dbg && j < 512) dbg[j * 4 + 1] = clock64();
        const uint32_t row0 = smem_u32(L.ell(smem, k));
        const uint32_t lw0 = smem_u32(L.leaf(smem, k)) - mbal[k] * 8;
        for (int b = top; b >= lo; b--, j++) {
            const uint32_t row = row0 + (uint32_t)(b - lo) * estride * 4;
            const uint32_t nxt = st0 + (((uint32_t)j + 1) & 1u) * n2 * 8;
            const uint32_t now = st0 + ((uint32_t)j & 1u) * n2 * 8;
            uint64_t *g = slab0 + (uint64_t)j * p.slab_words;
            uint64_t any = 0;
            if constexpr (NPL > 0) {
                // Thread t owns nodes t + i*NT: every address below is a
                // per-thread base plus a compile-time immediate. Three phases
                // so the NPL chains overlap: node words, "other" words, XOR +
                // stores. Decode is branch-free: idx*8 = e << 3 (flag bits
                // shift out), masks from sign-extending shifts of the flags.
                constexpr uint32_t NT = 32 * WPC;
                const uint32_t rowt = row + tid * 4, nowt = now + tid * 8;
                uint64_t *gt = g + tid;
                uint32_t e[NPL];
                uint64_t v[NPL];
#pragma unroll
                for (int i = 0; i < NPL; i++)
                    e[i] = (tid + i * NT < n2) ? lds_u32(rowt + i * NT * 4) : kSuccNone;
#pragma unroll
                for (int i = 0; i < NPL; i++)
                    v[i] = lds_u64(((e[i] & kSuccLeaf) ? lw0 : nxt) + (e[i] << 3));
#pragma unroll
                for (int i = 0; i < NPL; i++) {
                    const uint64_t mo = (uint64_t)((int64_t)((int32_t)(e[i] << 1)) >> 63);  // has other
                    const uint64_t ms = (uint64_t)((int64_t)((int32_t)e[i]) >> 63);         // NOT self
                    own[i] = (v[i] & mo) ^ (own[i] & ~ms);
                    if (tid + i * NT < n2) {
                        sts_u64(nowt + i * NT * 8, own[i]);
                        gt[i * NT] = own[i];
                    }
                    any |= own[i];
                }
            } else {  // generic: any number of nodes per thread, own values from shared memory
                for (uint32_t s = tid; s < n2; s += nthreads) {
                    const uint32_t e = lds_u32(row + s * 4);
                    const uint64_t v = lds_u64(((e & kSuccLeaf) ? lw0 : nxt) + (e << 3));
                    const uint64_t mo = (uint64_t)((int64_t)((int32_t)(e << 1)) >> 63);
                    const uint64_t ms = (uint64_t)((int64_t)((int32_t)e) >> 63);
                    const uint64_t acc = (v & mo) ^ (lds_u64(nxt + s * 8) & ~ms);
                    sts_u64(now + s * 8, acc);
                    g[s] = acc;
                    any |= acc;
                }
            }
            if (dbg && j < 512) dbg[j * 4 + 2] = clock64();
            bool live;
            if constexpr (one_warp) {
                live = __any_sync(0xffffffffu, any != 0);
                __syncwarp();
            } else {
                const bool wany = __any_sync(0xffffffffu, any != 0);
                const uint32_t vn = vslot == 2 ? 0 : vslot + 1;
                if ((tid & 31) == 0) {
                    if (wany) s_vote[vslot] = 1;
                    if (tid == 0) s_vote[vn] = 0;
                }
                trav::named_sync(trav::kBarNode, (int)nthreads);
                live = s_vote[vslot] != 0;
                vslot = vn;
            }
            if (dbg && j < 512) dbg[j * 4 + 3] = clock64();
            if (producer) s_live[j] = live;
            if ((!live && first_layer > b) || b <= b_lo) {  // zero with no leaves below, or shard start: done
                stopped = true;
                consumed = q + 1;
                j++;
                break;
            }
        }
        if (producer && !stopped && q + (int)L.NST < ngroups) issue(q + (int)L.NST, k), issued++;
        if (++k == L.NST) k = 0, par ^= 1;
    }
    // Slab headers: walked boundaries live / zero, the rest dead.
    __syncthreads();
    for (uint32_t x = tid; x < p.slab_stride; x += blockDim.x)
        hdrs[x] = (int)x < j ? make_uint4(circ_id, word, (uint32_t)(b_hi - (int)x), s_live[x] ? kSlabLive : kSlabZero)
                             : make_uint4(0, 0, 0, kSlabDead);
    // Drain groups staged below the stopping boundary (never consumed).
    if (producer)
        for (int x = consumed; x < issued; x++)
            mbar_wait(&full[(uint32_t)x % L.NST], (uint32_t)(x / (int)L.NST) & 1u);
}

// Circuits too wide for on-chip state (2n nodes x 2 buffers + staging beyond
// shared memory, about 4,800 qubits): the same walk with the state in global
// memory -- each boundary's column IS its slab (L2-resident), read back as
// the next boundary's successor values; ELLPACK rows and leaf words are read
// in place. One CTA per word, one block barrier (with the zero vote) per
// boundary. Slower than walk_kernel, but any width the workspace holds.
__global__ void __launch_bounds__(1024) walk_wide_kernel(__grid_constant__ const DevPlan p, TravCfg cfg) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ CircuitMeta s_meta;
    __shared__ uint32_t s_min_m, s_max_m, s_grp, s_circ;
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    if (tid == 0) {
        const uint32_t *circ_grp = arr<uint32_t>(p, p.lay.circ_grp);
        const uint32_t c = find_u32(circ_grp, p.tot.C, blockIdx.x);
        s_meta = arr<CircuitMeta>(p, p.lay.meta)[c];
        s_grp = blockIdx.x - circ_grp[c];
        s_circ = c;
        s_min_m = 0xFFFFFFFFu;
        s_max_m = 0;
    }
    __syncthreads();
    const CircuitMeta m = s_meta;
    const uint32_t word = s_grp, n2 = 2 * m.n, circ_id = s_circ;
    uint4 *hdrs = p.slab_hdr + (uint64_t)blockIdx.x * p.slab_stride;
    {  // measurement window of the word's detectors / observables (as walk_kernel)
        const uint32_t b0 = word * 64, b1 = min(b0 + 64, m.D + m.O);
        const uint32_t *doff = arr<uint32_t>(p, p.lay.det_off) + m.det_base;
        const uint32_t *dms = arr<uint32_t>(p, p.lay.det_meas);
        uint32_t lo = 0xFFFFFFFFu, hi = 0;
        for (uint32_t d = b0 + tid; d < min(b1, m.D); d += nt)
            for (uint32_t k = doff[d]; k < doff[d + 1]; k++) {
                lo = min(lo, dms[k]);
                hi = max(hi, dms[k]);
            }
        const uint32_t *ooff = arr<uint32_t>(p, p.lay.obs_off) + m.obs_base;
        const uint32_t *oms = arr<uint32_t>(p, p.lay.obs_meas);
        for (uint32_t b = max(b0, m.D); b < b1; b++)
            for (uint32_t k = ooff[b - m.D] + tid; k < ooff[b - m.D + 1]; k += nt) {
                lo = min(lo, oms[k]);
                hi = max(hi, oms[k]);
            }
        if (lo != 0xFFFFFFFFu) {
            atomicMin(&s_min_m, lo);
            atomicMax(&s_max_m, hi);
        }
    }
    __syncthreads();
    const uint32_t min_m = s_min_m, max_m = s_max_m;
    if (min_m == 0xFFFFFFFFu) {
        for (uint32_t x = tid; x < p.slab_stride; x += nt) hdrs[x] = make_uint4(0, 0, 0, kSlabDead);
        return;
    }
    const uint32_t lay_w = (cfg.max_l + 4) & ~3u;
    uint32_t *lay_meas = reinterpret_cast<uint32_t *>(smem);
    uint8_t *s_live = smem + (size_t)lay_w * 4;
    {
        const uint32_t *gm = arr<uint32_t>(p, p.lay.lay_meas) + m.layer_base;
        for (uint32_t i = tid; i <= m.l; i += nt) lay_meas[i] = gm[i];
    }
    __syncthreads();
    auto layer_of = [&](uint32_t mm) {
        uint32_t lo = 0, hi = m.l;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (lay_meas[mid] <= mm) lo = mid;
            else hi = mid;
        }
        return (int)lo;
    };
    const int first_layer = layer_of(min_m);
    const int b_hi = layer_of(max_m) - 1;
    const int b_lo = (int)min(p.shard_lo, 0x7FFFFFFFu);
    const uint32_t estride = ell_stride(m.n);
    const uint32_t *ell = p.ell + m.ell_base;
    const uint64_t *leaf = p.leaf + m.leaf_base + (uint64_t)word * leaf_stride(m.M);
    uint64_t *slab0 = p.slab + (uint64_t)blockIdx.x * p.slab_stride * p.slab_words;
    int j = 0;
    for (int b = b_hi; b >= b_lo && b >= 0; b--, j++) {
        const uint32_t *row = ell + (uint64_t)b * estride;
        const uint64_t *nxt = j ? slab0 + (uint64_t)(j - 1) * p.slab_words : nullptr;  // S_{b+1} (0 at the top)
        uint64_t *g = slab0 + (uint64_t)j * p.slab_words;
        uint64_t any = 0;
        for (uint32_t s = tid; s < n2; s += nt) {
            const uint32_t e = row[s], idx = e & kSuccIdx;
            uint64_t acc = (e & kSuccNotSelf) || !nxt ? 0 : nxt[s];
            if (e & kSuccOther) acc ^= (e & kSuccLeaf) ? leaf[idx] : (nxt ? nxt[idx] : 0);
            g[s] = acc;
            any |= acc;
        }
        const bool live = __syncthreads_or(any != 0) != 0;  // (also orders this column before the next reads it)
        if (tid == 0) s_live[j] = live;
        if ((!live && first_layer > b) || b <= b_lo) {
            j++;
            break;
        }
    }
    __syncthreads();
    for (uint32_t x = tid; x < p.slab_stride; x += nt)
        hdrs[x] = (int)x < j ? make_uint4(circ_id, word, (uint32_t)(b_hi - (int)x), s_live[x] ? kSlabLive : kSlabZero)
                             : make_uint4(0, 0, 0, kSlabDead);
}

// Files one signature record of `src`: word index and its nonzero bits.
__device__ __forceinline__ void put_record(const DevPlan &p, uint64_t src, uint32_t word, uint64_t bits) {
    const uint32_t j = atomicAdd(&p.cnt[src], 1u);
    if (j < p.K) {
        p.rbits[rec_at(p, src, j)] = bits;
        p.rtile[rec_at(p, src, j)] = word;
    } else {
        atomicMax(&p.hdr->record_overflow, j + 1);
    }
}

__global__ void __launch_bounds__(256) emit_kernel(__grid_constant__ const DevPlan p) {
    const uint64_t used = (uint64_t)p.tot.groups * p.slab_stride;
    const uint32_t level = p.tot.level;
    const CircuitMeta *meta = arr<CircuitMeta>(p, p.lay.meta);
    const uint32_t *lay_noise = arr<uint32_t>(p, p.lay.lay_noise);
    const uint64_t *noise = p.noise_words();
    // Noise ops at live boundaries: one CTA per slab.
    for (uint64_t sl = blockIdx.x; sl < used; sl += gridDim.x) {
        const uint4 h = p.slab_hdr[sl];
        if (h.w != kSlabLive) continue;
        if (h.z < p.shard_lo || h.z >= p.shard_hi) continue;  // fault-range shard: layer outside
        const CircuitMeta &m = meta[h.x];
        const uint64_t *st = p.slab + sl * p.slab_words;
        const uint32_t n0 = lay_noise[m.layer_base + h.z], n1 = lay_noise[m.layer_base + h.z + 1];
        for (uint32_t o = n0 + threadIdx.x; o < n1; o += blockDim.x) {
            const uint64_t wd = noise[o];
            const uint32_t kind = noise_kind(wd), q0 = noise_q0(wd);
            const uint64_t x0 = st[2 * q0], z0 = st[2 * q0 + 1];
            uint64_t x1 = 0, z1 = 0;
            if (kind == 3) {
                const uint32_t q1 = noise_q1(wd);
                x1 = st[2 * q1];
                z1 = st[2 * q1 + 1];
            }
            if (!(x0 | z0 | x1 | z1)) continue;
            const uint64_t src = m.src_base + p.nsrc[o];
            if (kind <= 1) {
                const uint64_t v = kind == 0 ? x0 : z0;
                if (v) put_record(p, src, h.y, v);
            } else if (kind == 2) {  // X, Z, then Y at L1+ (stepg.cpp:75-83)
                if (x0) put_record(p, src, h.y, x0);
                if (z0) put_record(p, src + 1, h.y, z0);
                if (level && (x0 ^ z0)) put_record(p, src + 2, h.y, x0 ^ z0);
            } else {
                const uint32_t nc = level == 0 ? 6 : level == 1 ? 10 : 15;
                for (uint32_t c = 0; c < nc; c++) {
                    const uint32_t mk = dep2_mask(c);
                    const uint64_t v = ((mk & 1) ? x0 : 0) ^ ((mk & 2) ? z0 : 0) ^ ((mk & 4) ? x1 : 0) ^
                                       ((mk & 8) ? z1 : 0);
                    if (v) put_record(p, src + c, h.y, v);
                }
            }
        }
    }
    // Measurement-flip sources (stepg.cpp:270-272): the signature of flip m is
    // leaf row m; per (measurement, word) the detector / observable holding
    // the word's lowest set bit files it, so each record is filed once.
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    const double *flip = arr<double>(p, p.lay.meas_flip);
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < p.tot.dets + p.tot.obss; t += nthreads) {
        uint32_t c, bit, k0, k1;
        const uint32_t *ms;
        if (t < p.tot.dets) {
            c = find_u32(arr<uint32_t>(p, p.lay.circ_det), p.tot.C, (uint32_t)t);
            bit = (uint32_t)t - arr<uint32_t>(p, p.lay.circ_det)[c];
            const uint32_t *off = arr<uint32_t>(p, p.lay.det_off) + meta[c].det_base;
            k0 = off[bit];
            k1 = off[bit + 1];
            ms = arr<uint32_t>(p, p.lay.det_meas);
        } else {
            const uint32_t to = (uint32_t)(t - p.tot.dets);
            c = find_u32(arr<uint32_t>(p, p.lay.circ_obs), p.tot.C, to);
            const uint32_t o = to - arr<uint32_t>(p, p.lay.circ_obs)[c];
            bit = meta[c].D + o;
            const uint32_t *off = arr<uint32_t>(p, p.lay.obs_off) + meta[c].obs_base;
            k0 = off[o];
            k1 = off[o + 1];
            ms = arr<uint32_t>(p, p.lay.obs_meas);
        }
        const CircuitMeta &m = meta[c];
        const uint64_t *row = p.leaf + m.leaf_base + (uint64_t)(bit >> 6) * leaf_stride(m.M);
        const uint32_t *lm = arr<uint32_t>(p, p.lay.lay_meas) + m.layer_base;
        const uint32_t m_lo = p.shard_lo <= m.l ? lm[p.shard_lo] : m.M;  // measurements of shard layers
        const uint32_t m_hi = p.shard_hi <= m.l ? lm[p.shard_hi] : m.M;
        for (uint32_t k = k0; k < k1; k++) {
            const uint32_t mm = ms[k];
            if (mm < m_lo || mm >= m_hi) continue;
            if (!(flip[m.meas_base + mm] > 0)) continue;
            const uint64_t v = row[mm];
            if (v && (uint32_t)__ffsll((long long)v) - 1 == (bit & 63)) put_record(p, m.src_base + m.src_noise + mm, bit >> 6, v);
        }
    }
}

}  // namespace walk

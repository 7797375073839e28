// gp_traverse.cuh -- K2: the Alg. 1 backward traversal (sm_100a), included by
// gp_kernels.cu.
//
// Replaces run_backward / run_subpass / update_cell (eec.cpp:64-122) and the
// per-source signature gather (eec.cpp:130-140; compile.cpp:34-39).
//
// One CTA owns one column group: T consecutive 64-bit detector words of one
// circuit (T = W when a whole circuit fits, so a CTA then owns every word of
// every source of its circuit). It walks the boundaries backwards keeping the
// group's columns of the class matrix for the live boundaries on chip. Warp
// roles, synchronised only through mbarriers (no CTA barrier per boundary):
//
//   warp 0        producer: one elected lane stages boundary b's ELLPACK slice,
//                 the next layer's leaf words and layer b's noise ops into a
//                 ring of NST shared buffers with cp.async.bulk (UBLKCP), up to
//                 NST-1 boundaries ahead;
//   node warps    the critical path: S_b[s] = XOR of S_{b+1} / leaf words named
//                 by node s's two successors, for all T words, into a ring of R
//                 state slots; one named barrier (with an OR-reduction for the
//                 all-zero test) per boundary among node warps only;
//   emit warps    trail the node warps by up to R-1 boundaries: every noise op
//                 placed at b XORs <= 4 base rows per component (the correlated
//                 slots of the reference are XORs of base rows) and emits only
//                 nonzero words (source, word, bits). With T = W the whole
//                 sparse signature is written by one thread without atomics.
//
// Time window: the group starts at the last layer holding one of its
// measurements and stops once its columns are zero below its first one.

namespace trav {

constexpr int kBarNode = 1, kBarEmit = 2;  // named barriers (0 = __syncthreads)

struct StageHdr {  // written by the producer into each stage
    uint32_t mb, me;          // local measurement range of layer b+1
    uint32_t n0, n1;          // global noise-op range of layer b
    uint32_t noise_shift;     // u64 words before op n0 in the staged noise slice
    uint32_t src_shift;       // u32 words before op n0 in the staged source-offset slice
    uint32_t leaf_shift[8];   // u64 words before meas mb in each staged leaf row
    uint32_t pad[2];          // keeps every staged buffer 16-byte aligned (cp.async.bulk)
};
static_assert(sizeof(StageHdr) % 16 == 0, "bulk-copy destinations must stay 16-byte aligned");

struct Dims {
    uint32_t T, R, NST, n2, ell_w, leaf_w, noise_w, src_w, lay_w, map_w, bkt_w, nzb_w;
    __host__ __device__ Dims(uint32_t t, uint32_t r, uint32_t nst, uint32_t max_n, uint32_t max_meas,
                             uint32_t max_noise, uint32_t max_l, uint32_t max_comp = 15, bool fuse_key = false)
        : T(t),
          R(r),
          NST(nst),
          n2(2 * max_n),
          ell_w(ell_stride(max_n)),
          leaf_w((max_meas + 3) & ~1u),
          noise_w((max_noise + 3) & ~1u),
          src_w((max_noise + 9) & ~3u),
          lay_w((max_l + 4) & ~3u),
          map_w((max_noise * max_comp + 8) & ~7u),
          bkt_w(fuse_key ? (64 * t + 4) & ~3u : 0),
          nzb_w(fuse_key ? ((2 * max_n + 31) / 32 + 3) & ~3u : 0) {}
    __host__ __device__ size_t ring_bytes() const { return (size_t)R * T * n2 * 8; }
    __host__ __device__ size_t stage_bytes() const {
        return sizeof(StageHdr) + (size_t)ell_w * 4 + ((size_t)T * leaf_w + noise_w) * 8 + (size_t)src_w * 4;
    }
    __host__ __device__ size_t total_bytes() const {
        return ring_bytes() + NST * stage_bytes() + (2 * NST + 2 * R) * 8 + (size_t)2 * lay_w * 4 + (size_t)bkt_w * 4 +
               (size_t)R * nzb_w * 4 + (size_t)map_w * 2 + 64;
    }
    __device__ uint64_t *slot(uint8_t *base, uint32_t r) const {
        return reinterpret_cast<uint64_t *>(base) + (size_t)r * T * n2;
    }
    __device__ uint8_t *stage(uint8_t *base, uint32_t k) const { return base + ring_bytes() + (size_t)k * stage_bytes(); }
    __device__ StageHdr *hdr(uint8_t *base, uint32_t k) const { return reinterpret_cast<StageHdr *>(stage(base, k)); }
    __device__ uint32_t *ell(uint8_t *base, uint32_t k) const {
        return reinterpret_cast<uint32_t *>(stage(base, k) + sizeof(StageHdr));
    }
    __device__ uint64_t *leaf(uint8_t *base, uint32_t k) const {
        return reinterpret_cast<uint64_t *>(ell(base, k) + ell_w);
    }
    __device__ uint64_t *noise(uint8_t *base, uint32_t k) const { return leaf(base, k) + (size_t)T * leaf_w; }
    __device__ uint32_t *src(uint8_t *base, uint32_t k) const {
        return reinterpret_cast<uint32_t *>(noise(base, k) + noise_w);
    }
    __device__ uint64_t *bars(uint8_t *base) const {
        return reinterpret_cast<uint64_t *>(base + ring_bytes() + NST * stage_bytes());
    }
    // Per-layer tables of the CTA's circuit (measurement / noise-op offsets).
    __device__ uint32_t *lay(uint8_t *base) const { return reinterpret_cast<uint32_t *>(bars(base) + 2 * NST + 2 * R); }
    // per-bucket source counts of the CTA's circuit (fused bucket keys)
    __device__ uint32_t *bkt(uint8_t *base) const { return lay(base) + 2 * lay_w; }
    // layer source -> op (source-major emission)
    // per state slot: one bit per base row, set when the row is nonzero (fused items)
    __device__ uint32_t *nzb(uint8_t *base, uint32_t r) const { return bkt(base) + bkt_w + r * nzb_w; }
    __device__ uint16_t *map(uint8_t *base) const {
        return reinterpret_cast<uint16_t *>(bkt(base) + bkt_w + R * nzb_w);
    }
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ bool named_or(int id, int nthreads, bool pred) {
    uint32_t out;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.ne.u32 p, %1, 0;\n\t"
        "bar.red.or.pred q, %2, %3, p;\n\t"
        "selp.u32 %0, 1, 0, q;\n\t}"
        : "=r"(out)
        : "r"((uint32_t)pred), "r"(id), "r"(nthreads)
        : "memory");
    return out != 0;
}

// Fused items (direct traversal: the CTA owns its circuit's every word):
// each nonempty source's reduce sort item (gp_reduce.cuh) is built here from
// the words in registers -- the probability from the flips / ptab3 -- and
// written to the circuit's item region in emission order (warp-aggregated
// slots: coalesced 32-byte stores) with its circuit-local bucket (first
// detector + 1). Records are written only for items whose key does not fit
// (the exact comparator reads them). At its end the CTA lists every bucket's
// items (boff[b] = {first, count}, iidx). This replaces the reduce's key and
// scatter passes (red::key_kernel, red::scatter_kernel) and their re-reads.
struct KeyCtx {
    uint32_t *sbkt;    // shared per-bucket counters (D + 1), or null: no fusion
    uint32_t *nitems;  // shared item counter of the circuit
    uint64_t src_base;
    uint32_t D;
};

template <int TM>
__device__ __forceinline__ void emit_item(const DevPlan &p, uint64_t src, uint32_t tw, const uint64_t (&v)[TM],
                                          const KeyCtx &kc, double prob) {
    uint64_t any = 0;
#pragma unroll
    for (int w = 0; w < TM; w++) any |= (uint32_t)w < tw ? v[w] : 0ull;
    const uint32_t am = __activemask(), lane = threadIdx.x & 31;
    const uint32_t want = __ballot_sync(am, any != 0);
    if (!want) return;
    const uint32_t leader = __ffs(want) - 1;
    uint32_t k = 0;
    if (lane == leader) k = atomicAdd(kc.nitems, (uint32_t)__popc(want));
    k = __shfl_sync(am, k, leader) + __popc(want & ((1u << lane) - 1));
    if (any == 0) return;
    uint32_t local;
    const red::Item it = red::item_of_words<TM>(v, tw, kc.D, prob, (uint32_t)src, p.force_collisions != 0, &local);
    if (!it.complete()) {  // the exact comparator reads this source's records
        uint32_t nz = 0;
#pragma unroll
        for (int w = 0; w < TM; w++) nz += ((uint32_t)w < tw && v[w] != 0);
        p.cnt[src] = nz;
        if (nz > p.K) {
            atomicMax(&p.hdr->record_overflow, nz);
        } else {
            uint32_t j = 0;
#pragma unroll
            for (int w = 0; w < TM; w++)
                if ((uint32_t)w < tw && v[w]) {
                    p.rbits[rec_at(p, src, j)] = v[w];
                    p.rtile[rec_at(p, src, j)] = (uint32_t)w;
                    j++;
                }
        }
    }
    const uint64_t at = kc.src_base + k;
    red::store_item(red::items_of(p) + at, it);
    p.ibkt[at] = (uint16_t)local;
    atomicAdd(&kc.sbkt[local], 1u);
}

// Writes one source's sparse signature words. `direct`: this CTA owns every
// word of the source (T == W), so the signature is written without atomics.
// Fused items: the source's sort item instead (prob is its probability).
template <int TM>
__device__ __forceinline__ void emit_source(const DevPlan &p, uint64_t src, uint32_t t0, uint32_t tw,
                                            const uint64_t (&v)[TM], bool direct, const KeyCtx &kc,
                                            double prob = 0.0) {
    if (kc.sbkt) {
        emit_item<TM>(p, src, tw, v, kc, prob);
        return;
    }
    uint32_t nz = 0;
#pragma unroll
    for (int w = 0; w < TM; w++) nz += ((uint32_t)w < tw && v[w] != 0);
    if (nz == 0) return;
    uint32_t j = direct ? 0u : atomicAdd(&p.cnt[src], nz);
    if (direct) p.cnt[src] = nz;
    if (j + nz > p.K) {
        atomicMax(&p.hdr->record_overflow, j + nz);
        return;
    }
#pragma unroll
    for (int w = 0; w < TM; w++)
        if ((uint32_t)w < tw && v[w]) {
            p.rbits[rec_at(p, src, j)] = v[w];
            p.rtile[rec_at(p, src, j)] = t0 + w;
            j++;
        }
}

// Warp-cooperative append into the record pool: lane-uniform chunk state,
// one warp scan per round, one chunk allocation (a returning atomic) per
// kPoolChunk records -- no per-record atomics on the traversal's path.
struct PoolWriter {
    uint32_t chunk;  // current chunk index (kPoolInvalid before the first)
    uint32_t fill;   // records used in the current chunk
};

__device__ __forceinline__ void pool_store(const DevPlan &p, uint32_t chunk, uint32_t pos, uint32_t src,
                                           uint32_t word, uint64_t bits) {
    if (chunk < p.pool_chunks_cap)
        p.pool[(size_t)chunk * kPoolChunk + pos] = make_uint4(src, word, (uint32_t)bits, (uint32_t)(bits >> 32));
}

// Every lane of the warp calls this in the same round; lane records are the
// components c with bit c of `mask` set: (src0 + c, word, bits[c]).
template <int NMAX>
__device__ __forceinline__ void pool_append(const DevPlan &p, PoolWriter &w, uint32_t lane, uint32_t mask,
                                            uint32_t src0, const uint64_t (&bits)[NMAX], uint32_t word) {
    const uint32_t n = __popc(mask);
    uint32_t incl = n;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= (uint32_t)d) incl += o;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) return;
    const uint32_t off = incl - n;
    uint32_t old = w.chunk, nxt = w.chunk;
    if (w.chunk == kPoolInvalid || w.fill + total > kPoolChunk) {
        uint32_t c = 0;
        if (lane == 0) {
            c = atomicAdd(&p.hdr->pool_chunks, 1u);
            if (c >= p.pool_chunks_cap) atomicAdd(&p.hdr->pool_overflow, 1u);
        }
        nxt = __shfl_sync(0xffffffffu, c, 0);
        if (w.chunk == kPoolInvalid) {  // first chunk: everything goes there
            old = nxt;
            w.fill = 0;
        }
    }
    uint32_t pos = w.fill + off;
#pragma unroll
    for (int x = 0; x < NMAX; x++)
        if (mask >> x & 1) {
            if (pos < kPoolChunk) pool_store(p, old, pos, src0 + x, word, bits[x]);
            else pool_store(p, nxt, pos - kPoolChunk, src0 + x, word, bits[x]);
            pos++;
        }
    const uint32_t end = w.fill + total;
    if (end >= kPoolChunk && old != nxt) {
        w.chunk = nxt;
        w.fill = end - kPoolChunk;
    } else {
        w.chunk = old;
        w.fill = end;
    }
}

// Pads the rest of the warp's last chunk with invalid records.
__device__ __forceinline__ void pool_close(const DevPlan &p, const PoolWriter &w, uint32_t lane) {
    if (w.chunk == kPoolInvalid) return;
    for (uint32_t pos = w.fill + lane; pos < kPoolChunk; pos += 32)
        pool_store(p, w.chunk, pos, kPoolInvalid, 0, 0);
}

template <int TM>
__global__ void __launch_bounds__(800, 1) traverse_kernel(__grid_constant__ const DevPlan p, TravCfg cfg) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ CircuitMeta s_meta;
    __shared__ uint32_t s_min_m, s_max_m;
    __shared__ volatile int s_stop;  // boundary where the node warps stopped early, or -1
    __shared__ int s_issued_lo;      // lowest boundary the producer staged
    __shared__ uint32_t s_grp;

    const Dims L(cfg.T, cfg.R, cfg.NST, cfg.max_n, cfg.max_layer_meas, cfg.max_layer_noise, cfg.max_l, cfg.max_comp,
                 cfg.fuse_key != 0);
    const uint32_t tid = threadIdx.x;
    const uint32_t warp = tid >> 5, lane = tid & 31;
    const uint32_t node_threads = cfg.node_warps * 32, emit_threads = cfg.emit_warps * 32;

    if (tid == 0) {
        const uint32_t *circ_grp = arr<uint32_t>(p, p.lay.circ_grp);
        const uint32_t c = find_u32(circ_grp, p.tot.C, blockIdx.x);
        s_meta = arr<CircuitMeta>(p, p.lay.meta)[c];
        s_grp = blockIdx.x - circ_grp[c];
        s_min_m = 0xFFFFFFFFu;
        s_max_m = 0;
        s_stop = -1;
        s_issued_lo = 0x7FFFFFFF;
    }
    __syncthreads();
    const CircuitMeta m = s_meta;
    const uint32_t t0 = s_grp * cfg.T, tw = min(cfg.T, m.W - t0);
    const uint32_t n2 = 2 * m.n;
    const bool direct = cfg.direct != 0;

    // Measurement window of the group's detectors / observables.
    {
        const uint32_t b0 = t0 * 64, b1 = min((t0 + tw) * 64, m.D + m.O);
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
    if (min_m == 0xFFFFFFFFu) return;  // every column of the group is zero

    const uint64_t *leaf = p.leaf + m.leaf_base;  // tile-major: leaf[t * M + m]
    // Layer tables staged on chip once: the producer reads them every boundary.
    uint32_t *lay_meas = L.lay(smem), *lay_noise = L.lay(smem) + L.lay_w;
    {
        const uint32_t *gm = arr<uint32_t>(p, p.lay.lay_meas) + m.layer_base;
        const uint32_t *gn = arr<uint32_t>(p, p.lay.lay_noise) + m.layer_base;
        for (uint32_t i = tid; i <= m.l; i += blockDim.x) {
            lay_meas[i] = gm[i];
            lay_noise[i] = gn[i];
        }
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

    uint64_t *bars = L.bars(smem);
    uint64_t *stage_full = bars, *stage_empty = bars + L.NST;
    uint64_t *state_full = bars + 2 * L.NST, *state_empty = bars + 2 * L.NST + L.R;
    if (tid == 0) {
        for (uint32_t k = 0; k < L.NST; k++) {
            mbar_init(&stage_full[k], 1);
            mbar_init(&stage_empty[k], 2);  // node warps + emit warps
        }
        for (uint32_t r = 0; r < L.R; r++) {
            mbar_init(&state_full[r], 1);
            mbar_init(&state_empty[r], 1);
        }
        mbar_fence_init();
    }
    {  // ring slot R-1 plays S_{b_hi+1} = 0 for the first boundary
        uint64_t *z = L.slot(smem, L.R - 1);
        for (uint32_t x = tid; x < L.T * n2; x += blockDim.x) z[x] = 0;
    }
    __shared__ uint32_t s_nitems;
    const KeyCtx kc{cfg.fuse_key && p.fused ? L.bkt(smem) : nullptr, &s_nitems, m.src_base, m.D};
    if (kc.sbkt)
        for (uint32_t x = tid; x <= m.D; x += blockDim.x) kc.sbkt[x] = 0;
    if (tid == 0) s_nitems = 0;
    __syncthreads();

    const uint32_t *ell = p.ell + m.ell_base;
    const uint32_t estride = ell_stride(m.n);
    const uint64_t *noise = p.noise_words();
    const uint32_t *nsrc = p.nsrc;

    if (warp == 0) {
        // ------------------------------------------------ producer (one lane)
        for (int j = 0; lane == 0 && b_hi - j >= 0; j++) {
            const int b = b_hi - j;
            const uint32_t k = (uint32_t)j % L.NST;
            if (j >= (int)L.NST) {  // wait until boundary b + NST released stage k
                const uint32_t par = (uint32_t)(j / (int)L.NST - 1) & 1u;
                bool ok = false;
                while (!(ok = mbar_try_wait_sleep(&stage_empty[k], par, 2000))) {  // (re-checks s_stop)
                    if (b < s_stop) break;
                    __nanosleep(4096);
                }
                if (!ok) break;
            }
            if (b < s_stop) break;  // below the node warps' stopping boundary: nothing to stage
            {
                StageHdr *h = L.hdr(smem, k);
                const uint32_t mb = lay_meas[b + 1], me = lay_meas[b + 2];
                const uint32_t n0 = lay_noise[b], n1 = lay_noise[b + 1];
                const uint64_t na = (uint64_t)(noise + n0) & ~15ull, ne = ((uint64_t)(noise + n1) + 15) & ~15ull;
                const uint64_t sa = (uint64_t)(nsrc + n0) & ~15ull, se = ((uint64_t)(nsrc + n1) + 15) & ~15ull;
                h->mb = mb;
                h->me = me;
                h->n0 = n0;
                h->n1 = n1;
                h->noise_shift = (uint32_t)(((uint64_t)(noise + n0) & 15ull) >> 3);
                h->src_shift = (uint32_t)(((uint64_t)(nsrc + n0) & 15ull) >> 2);
                uint32_t bytes = estride * 4;
                // leaf row slices [mb, me) of the tw words, 16-byte aligned
                // (addresses recomputed in the issue loop: no local arrays)
                auto leaf_slice = [&](uint32_t w, uint64_t *a) {
                    const uint64_t *row = leaf + (uint64_t)(t0 + w) * leaf_stride(m.M);
                    *a = (uint64_t)(row + mb) & ~15ull;
                    return me > mb ? (uint32_t)((((uint64_t)(row + me) + 15) & ~15ull) - *a) : 0u;
                };
                for (uint32_t w = 0; w < tw; w++) {
                    uint64_t a;
                    bytes += leaf_slice(w, &a);
                    h->leaf_shift[w] = (uint32_t)(((uint64_t)(leaf + (uint64_t)(t0 + w) * leaf_stride(m.M) + mb) & 15ull) >> 3);
                }
                const uint32_t nb = n1 > n0 ? (uint32_t)(ne - na) : 0, sb = n1 > n0 ? (uint32_t)(se - sa) : 0;
                bytes += nb + sb;
                fence_proxy_async();
                mbar_arrive_expect_tx(&stage_full[k], bytes);
                bulk_g2s(L.ell(smem, k), ell + (uint64_t)b * estride, estride * 4, &stage_full[k]);
                for (uint32_t w = 0; w < tw; w++) {
                    uint64_t a;
                    const uint32_t lb = leaf_slice(w, &a);
                    if (lb) bulk_g2s(L.leaf(smem, k) + (size_t)w * L.leaf_w, (const void *)a, lb, &stage_full[k]);
                }
                if (nb) bulk_g2s(L.noise(smem, k), (const void *)na, nb, &stage_full[k]);
                if (sb) bulk_g2s(L.src(smem, k), (const void *)sa, sb, &stage_full[k]);
            }
            s_issued_lo = b;
        }
        __syncwarp();
    } else if (warp <= cfg.node_warps) {
        // ------------------------------------------------ node warps (critical path)
        const uint32_t tn = tid - 32;
        for (int j = 0; b_hi - j >= 0; j++) {
            const int b = b_hi - j;
            const uint32_t k = (uint32_t)j % L.NST, r = (uint32_t)j % L.R;
            const uint32_t rp = (uint32_t)(j + (int)L.R - 1) % L.R;
            if (j >= (int)L.R) mbar_wait(&state_empty[r], (uint32_t)(j / (int)L.R - 1) & 1u);
            mbar_wait(&stage_full[k], (uint32_t)(j / (int)L.NST) & 1u);
            const StageHdr *h = L.hdr(smem, k);
            const uint32_t *s_ell = L.ell(smem, k);
            const uint64_t *s_leaf = L.leaf(smem, k);
            const uint64_t *nxt = L.slot(smem, rp);
            uint64_t *now = L.slot(smem, r);
            const uint32_t mb_al = h->mb & ~1u;  // leaf rows are 16-byte aligned: the slice starts there
            bool any = false;
            uint32_t *nzb = kc.sbkt ? L.nzb(smem, r) : nullptr;
            // (warp-uniform trip count: the row bitmap is a ballot per 32 rows)
            for (uint32_t s0 = tn - lane; s0 < ((cfg.debug & 2) ? 0 : n2); s0 += node_threads) {
                const uint32_t s = s0 + lane;
                bool row = false;
                if (s < n2) {
                    const uint32_t e = s_ell[s];
                    const uint32_t idx = e & kSuccIdx;
#pragma unroll
                    for (int w = 0; w < TM; w++) {
                        if ((uint32_t)w >= tw) break;
                        const uint64_t *nw = nxt + (size_t)w * n2;
                        const uint64_t *lw = s_leaf + (size_t)w * L.leaf_w - mb_al;
                        uint64_t acc = (e & kSuccNotSelf) ? 0 : nw[s];
                        if (e & kSuccOther) acc ^= (e & kSuccLeaf) ? lw[idx] : nw[idx];
                        now[(size_t)w * n2 + s] = acc;
                        row |= acc != 0;
                    }
                }
                any |= row;
                if (nzb) {
                    const uint32_t bits = __ballot_sync(0xffffffffu, row);
                    if (lane == 0) nzb[s0 >> 5] = bits;
                }
            }
            const bool live = named_or(kBarNode, (int)node_threads, any);
            const bool stop = !live && first_layer > b;  // zero here and no leaves below
            if (tn == 0) {
                if (stop) s_stop = b;
                mbar_arrive(&state_full[r]);
                mbar_arrive(&stage_empty[k]);
            }
            if (stop) break;
        }
    } else {
        // ------------------------------------------------ emit warps
        const uint32_t te = tid - 32 - node_threads;
        const uint32_t level = p.tot.level;
        {  // measurement-flip sources: their rows are the leaf rows (stepg.cpp:270-272)
            const double *flip = arr<double>(p, p.lay.meas_flip) + m.meas_base;
            const uint64_t src_flip = m.src_base + m.src_noise;
            for (uint32_t mm = min_m + te; mm <= max_m; mm += emit_threads) {
                if (!(flip[mm] > 0)) continue;
                uint64_t v[TM];
#pragma unroll
                for (int w = 0; w < TM; w++) v[w] = (uint32_t)w < tw ? leaf[(uint64_t)(t0 + w) * leaf_stride(m.M) + mm] : 0;
                emit_source<TM>(p, src_flip + mm, t0, tw, v, direct, kc, flip[mm]);
            }
        }
        PoolWriter pw{kPoolInvalid, 0};
        for (int j = 0; b_hi - j >= 0; j++) {
            const int b = b_hi - j;
            const uint32_t k = (uint32_t)j % L.NST, r = (uint32_t)j % L.R;
            mbar_wait(&state_full[r], (uint32_t)(j / (int)L.R) & 1u);
            mbar_wait(&stage_full[k], (uint32_t)(j / (int)L.NST) & 1u);
            const StageHdr *h = L.hdr(smem, k);
            const uint64_t *s_noise = L.noise(smem, k) + h->noise_shift;
            const uint32_t *s_src = L.src(smem, k) + h->src_shift;
            const uint64_t *now = L.slot(smem, r);
            const uint32_t nops = (cfg.debug & 1) ? 0 : h->n1 - h->n0;
            if (TM > 1 && direct && nops) {
                // Source-major: consecutive lanes take consecutive sources of
                // the layer (an op's components are consecutive sources), so
                // the signature stores of a warp are coalesced. Lane -> op
                // through a per-boundary source -> op map in shared memory,
                // built by the emit warps and ordered by the emit barrier
                // before it is read (and after the previous boundary's reads).
                const uint32_t sfirst = s_src[0];
                const uint32_t klast = noise_kind(s_noise[nops - 1]);
                const uint32_t ncl = klast <= 1 ? 1 : klast == 2 ? (level ? 3 : 2) : (level == 0 ? 6 : level == 1 ? 10 : 15);
                const uint32_t ns = s_src[nops - 1] + ncl - sfirst;
                uint16_t *smap = L.map(smem);  // layer source -> op, built per boundary
                for (uint32_t o = te; o < nops; o += emit_threads) {
                    const uint32_t kd = noise_kind(s_noise[o]);
                    const uint32_t nc = kd <= 1 ? 1 : kd == 2 ? (level ? 3 : 2) : (level == 0 ? 6 : level == 1 ? 10 : 15);
                    const uint32_t f = s_src[o] - sfirst;
                    for (uint32_t c = 0; c < nc; c++) smap[f + c] = (uint16_t)o;
                }
                named_sync(kBarEmit, (int)emit_threads);
                const uint32_t *nzb = kc.sbkt ? L.nzb(smem, r) : nullptr;  // (per boundary)
                for (uint32_t i = te; i < ns; i += emit_threads) {
                    const uint32_t ls = sfirst + i;
                    const uint32_t lo = smap[i];
                    const uint64_t wd = s_noise[lo];
                    const uint32_t kind = noise_kind(wd), c = ls - s_src[lo];
                    const uint32_t q0 = noise_q0(wd), q1 = noise_q1(wd);
                    uint32_t mk = kind == 0 ? 1u : kind == 1 ? 2u : kind == 2 ? (c == 0 ? 1u : c == 1 ? 2u : 3u)
                                                                              : dep2_mask(c);
                    if (kc.sbkt) {  // rows known to be zero are not read (most sources are empty)
                        const uint32_t r0 = 2 * q0, r1 = 2 * q1;
                        const uint32_t b0 = nzb[r0 >> 5] >> (r0 & 31), b1 = kind == 3 ? nzb[r1 >> 5] >> (r1 & 31) : 0u;
                        mk &= (b0 & 3u) | (b1 & 3u) << 2;
                    }
                    uint64_t v[TM];
#pragma unroll
                    for (int w = 0; w < TM; w++) {
                        uint64_t x = 0;
                        if ((uint32_t)w < tw) {
                            const uint64_t *row = now + (size_t)w * n2;
                            if (mk & 1) x ^= row[2 * q0];
                            if (mk & 2) x ^= row[2 * q0 + 1];
                            if (mk & 4) x ^= row[2 * q1];
                            if (mk & 8) x ^= row[2 * q1 + 1];
                        }
                        v[w] = x;
                    }
                    double pr = 0.0;
                    if (kc.sbkt)
                        pr = p.tot.wide_prob ? p.prob[m.src_base + ls]
                                             : p.ptab3[4 * noise_pidx(wd) + (kind == 2 ? 1 : kind == 3 ? 2 : 0)];
                    emit_source<TM>(p, m.src_base + ls, t0, tw, v, direct, kc, pr);
                }
            } else
            // Warp-uniform trip count (the pool path needs whole-warp rounds).
            for (uint32_t ob = te - lane; ob < nops; ob += emit_threads) {
                const uint32_t o = ob + lane;
                const bool act = o < nops;
                uint64_t wd = act ? s_noise[o] : 0;
                const uint32_t kind = act ? noise_kind(wd) : 0;
                const uint32_t q0 = noise_q0(wd), q1 = noise_q1(wd);
                const uint64_t src = m.src_base + (act ? s_src[o] : 0);
                if constexpr (TM == 1) {
                    if (!direct) {
                        // One word per source: build this op's nonzero component
                        // records and append them to the pool as a warp.
                        uint64_t a = 0, bz = 0, cx = 0, dz = 0;
                        if (act) {
                            a = now[2 * q0];
                            bz = now[2 * q0 + 1];
                            if (kind == 3) {
                                cx = now[2 * q1];
                                dz = now[2 * q1 + 1];
                            }
                        }
                        uint64_t rv[15];
                        uint32_t mask = 0;
                        if (act && (a | bz | cx | dz)) {
                            const uint32_t nc = kind <= 1 ? 1 : kind == 2 ? (level ? 3 : 2)
                                                                          : (level == 0 ? 6 : level == 1 ? 10 : 15);
#pragma unroll
                            for (int c = 0; c < 15; c++) {
                                uint32_t mk = dep2_mask(c);
                                if (kind == 0) mk = 1;
                                else if (kind == 1) mk = 2;
                                else if (kind == 2) mk = c == 0 ? 1 : c == 1 ? 2 : 3;
                                rv[c] = ((mk & 1) ? a : 0) ^ ((mk & 2) ? bz : 0) ^ ((mk & 4) ? cx : 0) ^
                                        ((mk & 8) ? dz : 0);
                                if ((uint32_t)c < nc && rv[c]) mask |= 1u << c;
                            }
                        }
                        pool_append<15>(p, pw, lane, mask, (uint32_t)src, rv, t0);
                        continue;
                    }
                }
                if (!act) continue;
                uint64_t x0[TM], z0[TM];
                uint64_t anyw = 0;
#pragma unroll
                for (int w = 0; w < TM; w++) {
                    x0[w] = (uint32_t)w < tw ? now[(size_t)w * n2 + 2 * q0] : 0;
                    z0[w] = (uint32_t)w < tw ? now[(size_t)w * n2 + 2 * q0 + 1] : 0;
                    anyw |= x0[w] | z0[w];
                }
                if (kind <= 1) {
                    if (anyw) emit_source<TM>(p, src, t0, tw, kind == 0 ? x0 : z0, direct, kc);
                } else if (kind == 2) {
                    if (!anyw) continue;
                    uint64_t y[TM];
#pragma unroll
                    for (int w = 0; w < TM; w++) y[w] = x0[w] ^ z0[w];
                    emit_source<TM>(p, src, t0, tw, x0, direct, kc);  // X, Z, then Y at L1+ (stepg.cpp:75-83)
                    emit_source<TM>(p, src + 1, t0, tw, z0, direct, kc);
                    if (level) emit_source<TM>(p, src + 2, t0, tw, y, direct, kc);
                } else {
                    // Component words are re-read from the on-chip state slot per
                    // component: keeps only T words live in registers.
                    const uint64_t *rx0 = now + 2 * q0, *rz0 = now + 2 * q0 + 1;
                    const uint64_t *rx1 = now + 2 * q1, *rz1 = now + 2 * q1 + 1;
#pragma unroll
                    for (int w = 0; w < TM; w++)
                        if ((uint32_t)w < tw) anyw |= rx1[(size_t)w * n2] | rz1[(size_t)w * n2];
                    if (!anyw) continue;
                    const uint32_t nc = level == 0 ? 6 : level == 1 ? 10 : 15;
                    for (uint32_t c = 0; c < nc; c++) {
                        const uint32_t mk = dep2_mask(c);
                        uint64_t v[TM];
#pragma unroll
                        for (int w = 0; w < TM; w++) {
                            const size_t o2 = (size_t)w * n2;
                            v[w] = (uint32_t)w >= tw ? 0
                                                     : ((mk & 1) ? rx0[o2] : 0) ^ ((mk & 2) ? rz0[o2] : 0) ^
                                                           ((mk & 4) ? rx1[o2] : 0) ^ ((mk & 8) ? rz1[o2] : 0);
                        }
                        emit_source<TM>(p, src + c, t0, tw, v, direct, kc);
                    }
                }
            }
            named_sync(kBarEmit, (int)emit_threads);
            if (te == 0) {
                mbar_arrive(&state_empty[r]);
                mbar_arrive(&stage_empty[k]);
            }
            if (b == s_stop) break;  // node warps stopped at b (their state_full arrive orders s_stop)
        }
        pool_close(p, pw, lane);
    }
    __syncthreads();
    if (kc.sbkt && !(cfg.debug & 8)) {  // list the circuit's buckets (the CTA owns all of them)
        const uint32_t nb = m.D + 1, ni = s_nitems;
        if (warp == 0) {  // exclusive scan of the counts, in place; boff = {first, count}
            uint32_t carry = 0;
            for (uint32_t x0 = 0; x0 < nb; x0 += 32) {
                const uint32_t x = x0 + lane;
                const uint32_t c = x < nb ? kc.sbkt[x] : 0;
                uint32_t inc = c;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
                    if (lane >= (uint32_t)d) inc += o;
                }
                const uint32_t off = carry + inc - c;
                if (x < nb) {
                    kc.sbkt[x] = off;
                    p.boff[m.bucket_base + x] = make_uint4((uint32_t)(m.src_base + off), c, 0, 0);
                }
                carry += __shfl_sync(0xffffffffu, inc, 31);
            }
        }
        __syncthreads();
        for (uint32_t k = tid; k < ni; k += blockDim.x) {
            const uint64_t at = m.src_base + k;
            const uint32_t pos = atomicAdd(&kc.sbkt[p.ibkt[at]], 1u);
            if (p.fused_move)
                red::store_item(reinterpret_cast<red::Item *>(p.items2) + m.src_base + pos,
                                red::load_item(red::items_of(p) + at));
            else
                p.iidx[m.src_base + pos] = (uint32_t)at;
        }
    }
    // Drain bulk copies staged below the stopping boundary (never consumed;
    // each is the latest use of its stage, so its phase parity is unambiguous).
    if (tid == 0)
        for (int b = s_issued_lo; b < s_stop; b++) {
            const int j = b_hi - b;
            mbar_wait(&stage_full[(uint32_t)j % L.NST], (uint32_t)(j / (int)L.NST) & 1u);
        }
}

}  // namespace trav

// gp_tiny.cuh -- the whole compile of one small circuit in ONE CTA (sm_100a),
// included by gp_kernels.cu. For circuits whose detectors and observables fit
// one 64-bit word (D + O <= 64: e.g. surface d = 3), the ~12 launches of the
// general pipeline cost more than their work (latency of the
// JIT case, compile.cpp:23-53). Everything lives in shared memory:
//
//   lowering   node words of every boundary (stepg.cpp:196-234, as
//              lower_kernel) and the leaf word of every measurement
//              (init_leaves, eec.cpp:40-58);
//   Alg. 1     S_b = successors of S_{b+1}, boundary by boundary from the last
//              (run_backward, eec.cpp:64-122), every S_b kept;
//   emission   every source's signature word from S_b (noise components as
//              XORs of base rows, as the traversal's emitters) or a leaf
//              (measurement flips), with its probability (p, p/3, p/15 by
//              IEEE division, stepg.cpp:66-103); empty signatures dropped;
//   reduce     identical signatures meet in a shared-memory hash table
//              (full-key compare); each group's member probabilities are
//              folded ascending from 0 (dem.cpp:97-106); the groups are
//              ranked in canonical order (dem.cpp:122-127);
//   output     straight into the mapped host arrays (no copy kernel).
// Source order is irrelevant to the result: a group's members are folded in
// value order and its signature is its key.

namespace tiny {

constexpr uint32_t kThreads = 1024;

// Shared memory: node words, leaves, every boundary's column, the items
// (signature, probability, table slot), the hash table (2 cap slots: key,
// count, member offset), the groups (slot, folded probability, order) and
// the members' probabilities; the layer tables are staged first.
struct Dims {
    uint32_t n2, l, M, cap;  // cap: items (power of two >= sources)
    __host__ __device__ static size_t a16(size_t x) { return (x + 15) & ~(size_t)15; }
    __host__ __device__ size_t lay_off() const { return 0; }
    __host__ __device__ size_t ell_off() const { return a16((size_t)2 * (l + 1) * 4); }
    __host__ __device__ size_t leaf_off() const { return ell_off() + a16((size_t)(l ? l - 1 : 0) * n2 * 4); }
    __host__ __device__ size_t state_off() const { return leaf_off() + a16((size_t)M * 8); }
    __host__ __device__ size_t sig_off() const { return state_off() + (size_t)l * n2 * 8; }
    __host__ __device__ size_t prob_off() const { return sig_off() + (size_t)cap * 8; }
    __host__ __device__ size_t slot_off() const { return prob_off() + (size_t)cap * 8; }
    __host__ __device__ size_t tkey_off() const { return slot_off() + (size_t)cap * 4; }  // 2 cap u64
    __host__ __device__ size_t tcnt_off() const { return tkey_off() + (size_t)cap * 16; }  // 2 cap u32
    __host__ __device__ size_t toff_off() const { return tcnt_off() + (size_t)cap * 8; }   // 2 cap u32
    __host__ __device__ size_t gslot_off() const { return toff_off() + (size_t)cap * 8; }  // cap u32
    __host__ __device__ size_t gord_off() const { return gslot_off() + (size_t)cap * 4; }  // cap u32
    __host__ __device__ size_t gprob_off() const { return gord_off() + (size_t)cap * 4; }  // cap f64
    __host__ __device__ size_t mp_off() const { return gprob_off() + (size_t)cap * 8; }    // cap f64
    __host__ __device__ size_t bytes() const { return mp_off() + (size_t)cap * 8; }
};

// Canonical order of two single-word signatures (D detectors, observables
// above): detector lists first, then observable lists (reduce's obs_cmp on
// each part: lexicographic order of ascending id lists).
__device__ __forceinline__ int sig_cmp1(uint64_t a, uint64_t b, uint64_t dm) {
    const int c = red::obs_cmp(a & dm, b & dm);
    return c ? c : red::obs_cmp(a & ~dm, b & ~dm);
}

__device__ __forceinline__ uint32_t block_excl_scan1(uint32_t v, uint32_t *warp_sums, uint32_t *total) {
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= (uint32_t)d) inc += o;
    }
    if (lane == 31) warp_sums[w] = inc;
    __syncthreads();
    if (w == 0) {
        const uint32_t x = lane < blockDim.x / 32 ? warp_sums[lane] : 0;
        uint32_t s = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, s, d);
            if (lane >= (uint32_t)d) s += o;
        }
        warp_sums[lane] = s - x;
        if (lane == 31) *total = s;
    }
    __syncthreads();
    const uint32_t r = warp_sums[w] + inc - v;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kThreads, 1) tiny_kernel(__grid_constant__ const DevPlan p) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint32_t s_cnt, s_ws[32], s_tot[4];
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    const CircuitMeta m = arr<CircuitMeta>(p, p.lay.meta)[0];
    const uint32_t n2 = 2 * m.n, l = m.l, D = m.D, O = m.O, level = p.tot.level;
    const Dims L{n2, l, m.M, p.tiny_cap};
    uint32_t *lay = reinterpret_cast<uint32_t *>(smem + L.lay_off());  // gate offsets | noise offsets
    uint32_t *ell = reinterpret_cast<uint32_t *>(smem + L.ell_off());
    uint64_t *leaf = reinterpret_cast<uint64_t *>(smem + L.leaf_off());
    uint64_t *S = reinterpret_cast<uint64_t *>(smem + L.state_off());  // S_b at b * n2
    uint64_t *sig = reinterpret_cast<uint64_t *>(smem + L.sig_off());
    double *prob = reinterpret_cast<double *>(smem + L.prob_off());
    const uint32_t *lay_gate = lay, *lay_noise = lay + l + 1;
    const bool narrow = p.tot.narrow != 0;
    const uint64_t *gates = arr<uint64_t>(p, p.lay.gates);
    const uint32_t *gates32 = arr<uint32_t>(p, p.lay.gates);
    const uint64_t *noise = arr<uint64_t>(p, p.lay.noise);
    const uint32_t *noise32 = arr<uint32_t>(p, p.lay.noise);

    // ---- the layer tables staged (the searches below read them), node words
    // idle, leaves cleared
    for (uint32_t x = tid; x <= l; x += nt) {
        lay[x] = arr<uint32_t>(p, p.lay.lay_gate)[m.layer_base + x];
        lay[l + 1 + x] = arr<uint32_t>(p, p.lay.lay_noise)[m.layer_base + x];
    }
    for (uint32_t x = tid; x < (l ? l - 1 : 0) * n2; x += nt) ell[x] = kEllIdle;
    for (uint32_t x = tid; x < m.M; x += nt) leaf[x] = 0;
    for (uint32_t x = tid; x < n2; x += nt) S[(size_t)(l - 1) * n2 + x] = 0;  // the last boundary: no successors
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    const uint32_t g_lo = lay_gate[1 < l ? 1 : l], g_hi = lay_gate[l];
    for (uint32_t g = g_lo + tid; g < g_hi; g += nt) {  // gates of layer i >= 1 fix boundary i - 1
        uint32_t li = 1, lo_ = 1, hi_ = l;
        while (hi_ - lo_ > 1) {
            const uint32_t mid = (lo_ + hi_) >> 1;
            if (lay_gate[mid] <= g) lo_ = mid;
            else hi_ = mid;
        }
        li = lo_;
        const uint64_t w = narrow ? widen_gate(gates32[g]) : gates[g];
        const uint32_t lo = (uint32_t)w, hi = (uint32_t)(w >> 32);
        const uint32_t q = lo & ((1u << kGateKindShift) - 1), kind = lo >> kGateKindShift;
        uint32_t *e = ell + (size_t)(li - 1) * n2;
        const uint32_t x = 2 * q, z = 2 * q + 1;
        switch (kind) {
            case 0:
                e[x] = kSuccNotSelf | kSuccOther | z;
                e[z] = kSuccNotSelf | kSuccOther | x;
                break;
            case 1:
                e[x] = kSuccOther | (2 * hi);
                e[z] = kEllIdle;
                e[2 * hi] = kEllIdle;
                e[2 * hi + 1] = kSuccOther | z;
                break;
            case 2:
                e[x] = kSuccNone;
                e[z] = kSuccNone;
                break;
            case 3:
                e[x] = kSuccOther | kSuccLeaf | hi;
                e[z] = kSuccNone;
                break;
            default:
                e[x] = kSuccNotSelf | kSuccOther | kSuccLeaf | hi;
                e[z] = kSuccNone;
                break;
        }
    }
    {
        const uint32_t *doff = arr<uint32_t>(p, p.lay.det_off) + m.det_base;
        const uint32_t *dms = arr<uint32_t>(p, p.lay.det_meas);
        const uint32_t *ooff = arr<uint32_t>(p, p.lay.obs_off) + m.obs_base;
        const uint32_t *oms = arr<uint32_t>(p, p.lay.obs_meas);
        for (uint32_t b = tid; b < D + O; b += nt) {
            const uint32_t k0 = b < D ? doff[b] : ooff[b - D], k1 = b < D ? doff[b + 1] : ooff[b - D + 1];
            for (uint32_t k = k0; k < k1; k++)
                atomicXor((unsigned long long *)&leaf[b < D ? dms[k] : oms[k]], 1ull << b);
        }
    }
    __syncthreads();
    // ---- Alg. 1: every boundary's column, from the last one down
    for (int b = (int)l - 2; b >= 0; b--) {
        const uint32_t *e = ell + (size_t)b * n2;
        const uint64_t *nx = S + (size_t)(b + 1) * n2;
        uint64_t *now = S + (size_t)b * n2;
        for (uint32_t s = tid; s < n2; s += nt) {
            const uint32_t w = e[s], idx = w & kSuccIdx;
            uint64_t acc = (w & kSuccNotSelf) ? 0 : nx[s];
            if (w & kSuccOther) acc ^= (w & kSuccLeaf) ? leaf[idx] : nx[idx];
            now[s] = acc;
        }
        __syncthreads();
    }
    // ---- emission: (signature, probability) of every nonempty source
    constexpr uint8_t kMask[15] = {4, 8, 1, 5, 2, 10, 12, 9, 3, 6, 13, 7, 15, 11, 14};
    const double *ptab = arr<double>(p, p.lay.prob_table);
    const double *nprob = arr<double>(p, p.lay.noise_prob);
    auto put = [&](uint64_t v, double pr) {
        if (!v) return;
        const uint32_t k = atomicAdd(&s_cnt, 1u);
        if (k < L.cap) {
            sig[k] = v;
            prob[k] = pr;
        }
    };
    const uint32_t n_lo = lay_noise[0], n_hi = lay_noise[l];
    for (uint32_t o = n_lo + tid; o < n_hi; o += nt) {
        uint32_t lo_ = 0, hi_ = l;  // layer of op o: lay_noise[b] <= o < lay_noise[b + 1]
        while (hi_ - lo_ > 1) {
            const uint32_t mid = (lo_ + hi_) >> 1;
            if (lay_noise[mid] <= o) lo_ = mid;
            else hi_ = mid;
        }
        const uint64_t *row = S + (size_t)lo_ * n2;
        const uint64_t w = narrow ? widen_noise(noise32[o]) : noise[o];
        const uint32_t kind = noise_kind(w), q0 = noise_q0(w), q1 = noise_q1(w);
        const double pr = p.tot.wide_prob ? nprob[o] : ptab[noise_pidx(w)];
        const double pe = kind == 2 ? __ddiv_rn(pr, 3.0) : kind == 3 ? __ddiv_rn(pr, 15.0) : pr;
        const uint64_t a = row[2 * q0], bz = row[2 * q0 + 1];
        if (kind <= 1) {
            put(kind == 0 ? a : bz, pe);
        } else if (kind == 2) {
            put(a, pe);
            put(bz, pe);
            if (level) put(a ^ bz, pe);
        } else {
            const uint64_t c = row[2 * q1], dz = row[2 * q1 + 1];
            const uint32_t nc = level == 0 ? 6 : level == 1 ? 10 : 15;
            for (uint32_t x = 0; x < nc; x++) {
                const uint32_t mk = kMask[x];
                put(((mk & 1) ? a : 0) ^ ((mk & 2) ? bz : 0) ^ ((mk & 4) ? c : 0) ^ ((mk & 8) ? dz : 0), pe);
            }
        }
    }
    {  // measurement flips: the leaf rows (stepg.cpp:270-272), flip > 0 only
        const double *flip = arr<double>(p, p.lay.meas_flip) + m.meas_base;
        for (uint32_t x = tid; x < m.M; x += nt)
            if (flip[x] > 0) put(leaf[x], flip[x]);
    }
    __syncthreads();
    const uint32_t n = s_cnt;
    if (n > L.cap) {  // (the host sized cap from the source count: cannot happen)
        if (tid == 0) atomicAdd(&p.hdr->bad_input, 1u);
        return;
    }
    // ---- groups: identical signatures meet in a shared-memory hash table
    const uint64_t dm = D >= 64 ? ~0ull : (1ull << D) - 1;
    const uint32_t tcap = 2 * L.cap;
    uint32_t *slot = reinterpret_cast<uint32_t *>(smem + L.slot_off());
    unsigned long long *tkey = reinterpret_cast<unsigned long long *>(smem + L.tkey_off());
    uint32_t *tcnt = reinterpret_cast<uint32_t *>(smem + L.tcnt_off());
    uint32_t *toff = reinterpret_cast<uint32_t *>(smem + L.toff_off());
    uint32_t *gslot = reinterpret_cast<uint32_t *>(smem + L.gslot_off());
    uint32_t *gord = reinterpret_cast<uint32_t *>(smem + L.gord_off());
    double *gprob = reinterpret_cast<double *>(smem + L.gprob_off());
    double *mp = reinterpret_cast<double *>(smem + L.mp_off());
    for (uint32_t x = tid; x < tcap; x += nt) {
        tkey[x] = 0;
        tcnt[x] = 0;
    }
    __syncthreads();
    for (uint32_t k = tid; k < n; k += nt) {  // (signatures are nonzero: 0 marks an empty slot)
        const unsigned long long v = sig[k];
        uint32_t h = (uint32_t)(mix64(v) >> 32) & (tcap - 1);
        while (true) {
            const unsigned long long cur = atomicCAS(&tkey[h], 0ull, v);
            if (cur == 0 || cur == v) break;
            h = (h + 1) & (tcap - 1);
        }
        slot[k] = h;
        atomicAdd(&tcnt[h], 1u);
    }
    __syncthreads();
    // slots -> groups (slot order) and member offsets: block scans over the table
    const uint32_t tper = (tcap + nt - 1) / nt, t0s = min(tcap, tid * tper), t1s = min(tcap, t0s + tper);
    uint32_t ng = 0, nm = 0;
    for (uint32_t h = t0s; h < t1s; h++) {
        ng += tcnt[h] != 0;
        nm += tcnt[h];
    }
    uint32_t g = block_excl_scan1(ng, s_ws, &s_tot[0]);
    uint32_t off = block_excl_scan1(nm, s_ws, &s_tot[1]);
    const uint32_t G = s_tot[0];
    for (uint32_t h = t0s; h < t1s; h++) {
        toff[h] = off;
        off += tcnt[h];
        if (tcnt[h]) gslot[g++] = h;
    }
    __syncthreads();
    for (uint32_t k = tid; k < n; k += nt) {  // members' probabilities, grouped
        const uint32_t h = slot[k];
        mp[toff[h] + atomicSub(&tcnt[h], 1u) - 1] = prob[k];
    }
    __syncthreads();
    for (uint32_t x = tid; x < G; x += nt) {  // sorted fold per group (dem.cpp:97-106)
        const uint32_t h = gslot[x];
        const uint32_t o = toff[h], e = h + 1 < tcap ? toff[h + 1] : n;
        gprob[x] = red::fold_sorted(mp, o, e);
    }
    // canonical order of the groups (dem.cpp:122-127): a rank per group (the
    // keys are distinct), or a bitonic sort of group indices for many groups
    if (G <= 2048) {
        for (uint32_t x = tid; x < G; x += nt) {
            const uint64_t me = tkey[gslot[x]];
            uint32_t r = 0;
            for (uint32_t y = 0; y < G; y++) r += sig_cmp1(tkey[gslot[y]], me, dm) < 0;
            gord[r] = x;
        }
    } else {
        uint32_t np2 = 1;
        while (np2 < G) np2 <<= 1;
        for (uint32_t x = tid; x < np2; x += nt) gord[x] = x;
        __syncthreads();
        auto before = [&](uint32_t a_, uint32_t b_) {  // group a_ strictly before b_ (indices >= G last)
            if (a_ >= G || b_ >= G) return a_ < G && b_ >= G;
            return sig_cmp1(tkey[gslot[a_]], tkey[gslot[b_]], dm) < 0;
        };
        for (uint32_t k = 2; k <= np2; k <<= 1)
            for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                for (uint32_t i = tid; i < np2; i += nt) {
                    const uint32_t x = i ^ j;
                    if (x > i) {
                        const uint32_t u = gord[i], v = gord[x];
                        if ((i & k) == 0 ? before(v, u) : before(u, v)) {
                            gord[i] = v;
                            gord[x] = u;
                        }
                    }
                }
                __syncthreads();
            }
    }
    __syncthreads();
    // ---- edges in canonical order: id offsets by block scans, then written
    const uint64_t bE = p.base_in[0], bD = p.base_in[1], bO = p.base_in[2];
    const uint32_t gper = (G + nt - 1) / nt, g0 = min(G, tid * gper), g1 = min(G, g0 + gper);
    uint32_t nd = 0, no = 0;
    for (uint32_t r = g0; r < g1; r++) {
        const uint64_t v = tkey[gslot[gord[r]]];
        nd += __popcll(v & dm);
        no += __popcll(v & ~dm);
    }
    uint32_t dd = block_excl_scan1(nd, s_ws, &s_tot[1]);
    uint32_t oo = block_excl_scan1(no, s_ws, &s_tot[2]);
    const uint32_t E = G, ND = s_tot[1], NO = s_tot[2];
    const bool fits = E <= p.e_cap && ND <= p.ids_cap && NO <= p.ids_cap;
    auto &hm = p.hmap;
    if (fits)
        for (uint32_t r = g0; r < g1; r++) {
            const uint32_t x = gord[r];
            const uint64_t v = tkey[gslot[x]];
            hm.det_off[r] = (uint32_t)(bD + dd);
            hm.obs_off[r] = (uint32_t)(bO + oo);
            hm.probs[r] = gprob[x];
            for (uint64_t y = v & dm; y; y &= y - 1) hm.det_ids[dd++] = (uint32_t)__ffsll((long long)y) - 1;
            for (uint64_t y = v & ~dm; y; y &= y - 1) hm.obs_ids[oo++] = (uint32_t)__ffsll((long long)y) - 1 - D;
        }
    if (tid == 0) {
        DeviceHeader h{};
        if (fits) {
            h.num_edges = E;
            h.num_det_ids = ND;
            h.num_obs_ids = NO;
            hm.det_off[E] = (uint32_t)(bD + ND);
            hm.obs_off[E] = (uint32_t)(bO + NO);
            hm.edge_off[0] = bE;
            hm.edge_off[1] = bE + E;
        } else {
            h.num_det_ids = 0xFFFFFFFFu;  // capacity overflow marker: re-run larger
        }
        *p.hdr = h;
        *p.hdr_out = h;
        __threadfence_system();
        *hm.hdr = h;
    }
}

}  // namespace tiny

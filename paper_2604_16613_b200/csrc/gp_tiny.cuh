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

constexpr uint32_t kThreads = 1024;  // (launched with up to this many; see enqueue_pipeline)

// Shared memory: node words, leaves, every boundary's column, the items
// (signature, probability, table slot), the hash table (2 cap slots: key,
// count, member offset), the groups (slot, folded probability, order) and
// the members' probabilities; the layer tables are staged first.
struct Dims {
    uint32_t n2, l, M, cap;  // cap: items (power of two >= sources)
    uint32_t head;           // bytes of the staged image head (lay tables, detector / observable lists, probabilities)
    __host__ __device__ static size_t a16(size_t x) { return (x + 15) & ~(size_t)15; }
    __host__ __device__ size_t lay_off() const { return 0; }
    __host__ __device__ size_t ell_off() const { return a16(head); }
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
    __host__ __device__ size_t mp2_off() const { return mp_off() + (size_t)cap * 8; }    // cap f64
    __host__ __device__ size_t bytes() const { return mp2_off() + (size_t)cap * 8; }
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

// Staged image head: u32 gate offsets | noise offsets | detector offsets |
// observable offsets | detector measurements | observable measurements, then
// f64 probabilities [P] (G / N / M / wide: room for staged gate and noise
// words, flips and per-op probabilities -- measured slower than reading them
// in place, so the kernel stages none).
struct Head {
    uint32_t u32, P, G, N, M, wide;
    __host__ __device__ size_t f64_off() const { return ((size_t)u32 * 4 + 7) & ~(size_t)7; }
    __host__ __device__ size_t gate_off() const { return f64_off() + (size_t)P * 8; }
    __host__ __device__ size_t noise_off() const { return gate_off() + (size_t)G * 8; }
    __host__ __device__ size_t flip_off() const { return noise_off() + (size_t)N * 8; }
    __host__ __device__ size_t nprob_off() const { return flip_off() + (size_t)M * 8; }
    __host__ __device__ size_t bytes() const { return nprob_off() + (wide ? (size_t)N * 8 : 0); }
};
__host__ __device__ inline Head head_of(uint32_t l, uint32_t D, uint32_t O, uint32_t DE, uint32_t OE, uint32_t P,
                                        uint32_t G, uint32_t N, uint32_t M, bool wide) {
    return Head{2 * (l + 1) + D + 1 + O + 1 + DE + OE, wide ? 0 : P, G, N, M, wide ? 1u : 0u};
}

__device__ __forceinline__ uint64_t gtime() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(kThreads, 1) tiny_kernel(__grid_constant__ const DevPlan p) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint32_t nmark = 0;  // experiments (p.dbg): phase timestamps of thread 0
    auto mark = [&]() {
        if (p.dbg && threadIdx.x == 0) p.dbg[nmark] = gtime();
        nmark++;
    };
    mark();
    __shared__ uint32_t s_cnt, s_ws[32], s_tot[4];
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    const CircuitMeta &m = p.tiny_meta;  // (in the parameters: no dependent load at entry)
    const uint32_t n2 = 2 * m.n, l = m.l, D = m.D, O = m.O, level = p.tot.level;
    const uint32_t DE = (uint32_t)p.tot.det_entries, OE = (uint32_t)p.tot.obs_entries;
    const uint32_t P = p.tot.wide_prob ? 0 : p.tot.prob_table_n;
    const bool wide = p.tot.wide_prob != 0;
    const Head H = head_of(l, D, O, DE, OE, P, 0, 0, 0, wide);  // (gate / noise words and flips: read in place)
    const Dims L{n2, l, m.M, p.tiny_cap, (uint32_t)H.bytes()};
    // staged head: gate offsets | noise offsets | detector offsets | observable
    // offsets | detector measurements | observable measurements ; probabilities
    uint32_t *lay = reinterpret_cast<uint32_t *>(smem + L.lay_off());
    uint32_t *s_doff = lay + 2 * (l + 1), *s_ooff = s_doff + D + 1, *s_dms = s_ooff + O + 1, *s_oms = s_dms + DE;
    double *s_ptab = reinterpret_cast<double *>(smem + H.f64_off());
    uint32_t *ell = reinterpret_cast<uint32_t *>(smem + L.ell_off());
    uint64_t *leaf = reinterpret_cast<uint64_t *>(smem + L.leaf_off());
    uint64_t *S = reinterpret_cast<uint64_t *>(smem + L.state_off());  // S_b at b * n2
    uint64_t *sig = reinterpret_cast<uint64_t *>(smem + L.sig_off());
    double *prob = reinterpret_cast<double *>(smem + L.prob_off());
    const uint32_t *lay_gate = lay, *lay_noise = lay + l + 1;
    const bool narrow = p.tot.narrow != 0;

    // ---- one round of independent loads (the image may be pinned host
    // memory, read over PCIe): this thread's share of the head -- layer
    // tables, detector / observable lists, probability table -- and its first
    // gate word, noise word and measurement flip
    const uint32_t NGt = (uint32_t)p.tot.gates, NNt = (uint32_t)p.tot.noise;
    const uint64_t gw0 = tid < NGt ? (narrow ? widen_gate(arr<uint32_t>(p, p.lay.gates)[m.gate_base + tid])
                                             : arr<uint64_t>(p, p.lay.gates)[m.gate_base + tid])
                                   : 0;
    const uint64_t nw0 = tid < NNt ? (narrow ? widen_noise(arr<uint32_t>(p, p.lay.noise)[m.noise_base + tid])
                                             : arr<uint64_t>(p, p.lay.noise)[m.noise_base + tid])
                                   : 0;
    const double f0 = tid < m.M ? arr<double>(p, p.lay.meas_flip)[m.meas_base + tid] : 0.0;
    {
        const uint32_t nl = l + 1, nd = D + 1, no = O + 1;
        const uint32_t hu = 2 * nl + nd + no + DE + OE;  // u32 words of the head, then P doubles
        for (uint32_t u = tid; u < hu + P; u += nt) {
            if (u >= hu) {
                s_ptab[u - hu] = arr<double>(p, p.lay.prob_table)[u - hu];
                continue;
            }
            uint32_t x = u, v;
            if (x < nl) v = arr<uint32_t>(p, p.lay.lay_gate)[m.layer_base + x];
            else if ((x -= nl) < nl) v = arr<uint32_t>(p, p.lay.lay_noise)[m.layer_base + x];
            else if ((x -= nl) < nd) v = arr<uint32_t>(p, p.lay.det_off)[m.det_base + x] - (uint32_t)m.det_entry_base;
            else if ((x -= nd) < no) v = arr<uint32_t>(p, p.lay.obs_off)[m.obs_base + x] - (uint32_t)m.obs_entry_base;
            else if ((x -= no) < DE) v = arr<uint32_t>(p, p.lay.det_meas)[m.det_entry_base + x];
            else v = arr<uint32_t>(p, p.lay.obs_meas)[m.obs_entry_base + x - DE];
            lay[u] = v;  // (lay, s_doff, s_ooff, s_dms, s_oms are consecutive)
        }
    }
    for (uint32_t x = tid; x < (l ? l - 1 : 0) * n2; x += nt) ell[x] = kEllIdle;
    for (uint32_t x = tid; x < m.M; x += nt) leaf[x] = 0;
    for (uint32_t x = tid; x < n2; x += nt) S[(size_t)(l - 1) * n2 + x] = 0;  // the last boundary: no successors
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    mark();
    for (uint32_t gi = tid; gi < NGt; gi += nt) {  // gates of layer i >= 1 fix boundary i - 1
        const uint32_t g = (uint32_t)m.gate_base + gi;
        uint32_t lo_ = 0, hi_ = l;  // layer of gate g
        while (hi_ - lo_ > 1) {
            const uint32_t mid = (lo_ + hi_) >> 1;
            if (lay_gate[mid] <= g) lo_ = mid;
            else hi_ = mid;
        }
        const uint32_t li = lo_;
        if (li == 0) continue;  // (no boundary before layer 0)
        const uint64_t w = gi == tid ? gw0
                                     : narrow ? widen_gate(arr<uint32_t>(p, p.lay.gates)[g]) : arr<uint64_t>(p, p.lay.gates)[g];
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
    for (uint32_t b = tid; b < D + O; b += nt) {  // leaves (from the staged lists)
        const uint32_t k0 = b < D ? s_doff[b] : s_ooff[b - D], k1 = b < D ? s_doff[b + 1] : s_ooff[b - D + 1];
        for (uint32_t k = k0; k < k1; k++) atomicXor((unsigned long long *)&leaf[b < D ? s_dms[k] : s_oms[k]], 1ull << b);
    }
    // the emission's inputs of this thread's first noise op (its word came in
    // the first round)
    const double *ptab = s_ptab;
    const double *nprob = arr<double>(p, p.lay.noise_prob);
    const double *flip = arr<double>(p, p.lay.meas_flip) + m.meas_base;
    const uint32_t n_lo = lay_noise[0], n_hi = lay_noise[l];
    struct Op {
        uint32_t kind, q0, q1, b;
        double pe;
    };
    auto load_op = [&](uint32_t o) {
        uint32_t lo_ = 0, hi_ = l;  // layer of op o: lay_noise[b] <= o < lay_noise[b + 1]
        while (hi_ - lo_ > 1) {
            const uint32_t mid = (lo_ + hi_) >> 1;
            if (lay_noise[mid] <= o) lo_ = mid;
            else hi_ = mid;
        }
        const uint64_t w = o == n_lo + tid ? nw0
                                           : narrow ? widen_noise(arr<uint32_t>(p, p.lay.noise)[o])
                                                    : arr<uint64_t>(p, p.lay.noise)[o];
        const uint32_t kind = noise_kind(w);
        const double pr = wide ? nprob[o] : ptab[noise_pidx(w)];
        return Op{kind, noise_q0(w), noise_q1(w), lo_,
                  kind == 2 ? __ddiv_rn(pr, 3.0) : kind == 3 ? __ddiv_rn(pr, 15.0) : pr};
    };
    const Op op0 = n_lo + tid < n_hi ? load_op(n_lo + tid) : Op{0, 0, 0, 0, 0.0};
    __syncthreads();
    mark();
    // ---- Alg. 1: every boundary's column, from the last one down
    {  // (only the warps holding nodes walk, on a named barrier of their own)
        const uint32_t wt = min(nt, (n2 + 31) & ~31u);
        if (tid < wt)
            for (int b = (int)l - 2; b >= 0; b--) {
                const uint32_t *e = ell + (size_t)b * n2;
                const uint64_t *nx = S + (size_t)(b + 1) * n2;
                uint64_t *now = S + (size_t)b * n2;
                for (uint32_t s = tid; s < n2; s += wt) {
                    const uint32_t w = e[s], idx = w & kSuccIdx;
                    uint64_t acc = (w & kSuccNotSelf) ? 0 : nx[s];
                    if (w & kSuccOther) acc ^= (w & kSuccLeaf) ? leaf[idx] : nx[idx];
                    now[s] = acc;
                }
                if (wt > 32) asm volatile("bar.sync 1, %0;" ::"r"(wt) : "memory");
                else __syncwarp();
            }
        __syncthreads();
    }
    mark();
    // ---- emission: (signature, probability) of every nonempty source; a
    // counting pass and a block scan give each thread its item slots
    auto each = [&](auto &&f) {  // f(signature, probability) for every source of this thread
        for (uint32_t o = n_lo + tid; o < n_hi; o += nt) {
            const Op op = o == n_lo + tid ? op0 : load_op(o);
            const uint64_t *row = S + (size_t)op.b * n2;
            const uint64_t a = row[2 * op.q0], bz = row[2 * op.q0 + 1];
            if (op.kind <= 1) {
                f(op.kind == 0 ? a : bz, op.pe);
            } else if (op.kind == 2) {
                f(a, op.pe);
                f(bz, op.pe);
                if (level) f(a ^ bz, op.pe);
            } else {
                const uint64_t c = row[2 * op.q1], dz = row[2 * op.q1 + 1];
                const uint32_t nc = level == 0 ? 6 : level == 1 ? 10 : 15;
                for (uint32_t x = 0; x < nc; x++) {
                    const uint32_t mk = dep2_mask(x);
                    f(((mk & 1) ? a : 0) ^ ((mk & 2) ? bz : 0) ^ ((mk & 4) ? c : 0) ^ ((mk & 8) ? dz : 0), op.pe);
                }
            }
        }
        // measurement flips: the leaf rows (stepg.cpp:270-272), flip > 0 only
        for (uint32_t x = tid; x < m.M; x += nt) {
            const double fx = x == tid ? f0 : flip[x];
            if (fx > 0) f(leaf[x], fx);
        }
    };
    uint32_t mine = 0;
    each([&](uint64_t v, double) { mine += v != 0; });
    uint32_t k = block_excl_scan1(mine, s_ws, &s_tot[3]);
    if (s_tot[3] <= L.cap)
        each([&](uint64_t v, double pr) {
            if (v) {
                sig[k] = v;
                prob[k] = pr;
                k++;
            }
        });
    if (tid == 0) s_cnt = s_tot[3];
    __syncthreads();
    mark();
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
    mark();
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
    mark();
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
    mark();
    uint32_t *mpos = reinterpret_cast<uint32_t *>(sig);  // (signatures live in the table from here on)
    double *mp2 = reinterpret_cast<double *>(smem + L.mp2_off());
    for (uint32_t k = tid; k < n; k += nt) {  // members' probabilities, grouped (any order)
        const uint32_t h = slot[k];
        const uint32_t pos = toff[h] + atomicSub(&tcnt[h], 1u) - 1;
        mp[pos] = prob[k];
        mpos[k] = pos;
    }
    __syncthreads();
    // every member's rank in its group by (value, position): the group sorted
    // ascending in mp2 in one parallel step (a group holding a NaN is flagged
    // and sorted by its folding thread instead)
    for (uint32_t k = tid; k < n; k += nt) {
        const uint32_t h = slot[k], me = mpos[k];
        const uint32_t o = toff[h], e = h + 1 < tcap ? toff[h + 1] : n;
        const double v = prob[k];
        if (v != v) {
            tcnt[h] = 1;
            continue;
        }
        uint32_t r = 0;
        for (uint32_t j = o; j < e; j++) {
            const double w = mp[j];
            r += (w < v) || (w == v && j < me);
        }
        mp2[o + r] = v;
    }
    __syncthreads();
    mark();
    for (uint32_t x = tid; x < G; x += nt) {  // ascending fold per group from 0 (dem.cpp:97-106)
        const uint32_t h = gslot[x];
        const uint32_t o = toff[h], e = h + 1 < tcap ? toff[h + 1] : n;
        if (tcnt[h]) {
            gprob[x] = red::fold_sorted(mp, o, e);
        } else {
            double acc = 0.0;
            for (uint32_t j = o; j < e; j++) acc = merge_prob(acc, mp2[j]);
            gprob[x] = acc;
        }
    }
    __syncthreads();
    mark();
    // canonical order of the groups (dem.cpp:122-127): a rank per group (the
    // keys are distinct), or a bitonic sort of group indices for many groups
    uint64_t *gsig = reinterpret_cast<uint64_t *>(prob);  // (member probabilities are folded: reuse)
    for (uint32_t x = tid; x < G; x += nt) gsig[x] = tkey[gslot[x]];
    __syncthreads();
    if (G <= 2048) {
        // tpg threads (a power of two <= 32, lanes of one warp) share a group's
        // comparisons; the block's loop bound is uniform (warp shuffles)
        uint32_t tpg = 1;
        while (tpg < 32 && tpg * 2 * G <= nt) tpg *= 2;
        const uint32_t per_round = nt / tpg, j = tid % tpg;
        for (uint32_t xb = 0; xb < G; xb += per_round) {
            const uint32_t x = xb + tid / tpg;
            uint32_t r = 0;
            if (x < G) {
                const uint64_t me = gsig[x];
                for (uint32_t y = j; y < G; y += tpg) r += sig_cmp1(gsig[y], me, dm) < 0;
            }
            for (uint32_t d = tpg >> 1; d > 0; d >>= 1) r += __shfl_xor_sync(0xffffffffu, r, d);
            if (x < G && j == 0) gord[r] = x;
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
    mark();
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
    mark();
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
    mark();
}

}  // namespace tiny

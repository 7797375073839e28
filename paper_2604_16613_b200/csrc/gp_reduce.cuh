// gp_reduce.cuh -- K3 reduce (sm_100a), included by gp_kernels.cu.
//
// Replaces reduce_packed (dem.cpp:57-142): group identical signatures, fold
// each group's probabilities in ascending order from 0 (dem.cpp:97-106), and
// emit the groups in the canonical order (dem.cpp:122-127).
//
// The reference hashes dense W-word signatures, sorts them by (hash, words)
// and then sorts the groups again for the canonical order. Here one
// observation removes both global sorts: identical signatures share their
// first id, and the canonical order is lexicographic with the first id most
// significant. So sources are bucketed by (circuit, first detector) with a
// counting sort (key_kernel, a bucket scan, scatter_kernel), and each bucket
// is then sorted, grouped and folded on chip (bucket_kernel). A bucket scan
// gives every group its output slot (write_kernel).
//
// Canonical order as a sequence: a signature with detector ids d0<d1<... and
// observable ids o0<o1<... is the sequence  d0+1, d1+1, ..., 0, o0+1, ..., 0
// (then 0 forever). std::vector's lexicographic (dets, obs) compare -- a
// prefix sorts first -- is exactly the lexicographic compare of these
// sequences. seq[0] picks the bucket; seq[1..4] form a 128-bit sort key that
// decides almost every compare; the rest is compared exactly (full records)
// only when two keys tie, so distinct signatures never merge
// (dem.cpp:73-78, test_dem.cpp:94-101).

#include <type_traits>

namespace red {

constexpr uint32_t kBucketThreads = 128, kWarpItems = 256;  // bucket_kernel: a warp groups up to kWarpItems


// Slots of source s's records sorted by word (insertion sort, n <= 16).
__device__ __forceinline__ uint32_t sig_order(const DevPlan &p, uint64_t s, uint32_t n, uint8_t *ord) {
    uint32_t tile[16];
    for (uint32_t x = 0; x < n; x++) {
        const uint32_t t = p.rtile[rec_at(p, s, x)];
        uint32_t b = x;
        while (b > 0 && tile[b - 1] > t) {
            tile[b] = tile[b - 1];
            ord[b] = ord[b - 1];
            b--;
        }
        tile[b] = t;
        ord[b] = (uint8_t)x;
    }
    return n;
}

// Lazy generator of the canonical sequence of one signature (holds only the
// record arrays it reads: no pointer to the kernel's parameter block).
struct SeqIt {
    const uint32_t *rtile;
    const uint64_t *rbits;
    uint64_t stride;          // slot-major records: slot j at j * stride
    uint32_t n, D, r, phase;  // phase 0: detectors, 1: observables, 2: done
    uint64_t bits;
    uint32_t tile;
    uint8_t ord[16];

    __device__ void init(const DevPlan &pl, uint64_t src, uint32_t d) {
        rtile = pl.rtile + src;
        rbits = pl.rbits + src;
        stride = pl.tot.sources;
        D = d;
        n = min(pl.cnt[src], 16u);
        sig_order(pl, src, n, ord);
        phase = 0;
        r = 0;
        load();
    }
    __device__ uint64_t mask(uint32_t t) const {  // bits of word t in the current phase
        const uint32_t b0 = t * 64;
        uint64_t dm;
        if (b0 + 64 <= D) dm = ~0ull;
        else if (b0 >= D) dm = 0;
        else dm = (1ull << (D - b0)) - 1;
        return phase == 0 ? dm : ~dm;
    }
    __device__ void load() {
        bits = 0;
        while (r < n) {
            const uint32_t slot = ord[r];
            tile = rtile[slot * stride];
            bits = rbits[slot * stride] & mask(tile);
            if (bits) return;
            r++;
        }
    }
    __device__ uint32_t next() {
        if (phase == 2) return 0;
        if (r >= n) {  // end of this phase: separator
            phase++;
            r = 0;
            if (phase == 1) load();
            return 0;
        }
        const uint32_t b = (uint32_t)__ffsll((long long)bits) - 1;
        const uint32_t id = tile * 64 + b;
        bits &= bits - 1;
        if (!bits) {
            r++;
            load();
        }
        return phase == 0 ? id + 1 : id - D + 1;
    }
};

// Exact canonical compare of two signatures (-1, 0, 1).
__device__ __forceinline__ int seq_cmp(const DevPlan &p, uint64_t a, uint64_t b, uint32_t D) {
    SeqIt x, y;
    x.init(p, a, D);
    y.init(p, b, D);
    while (true) {
        const uint32_t u = x.next(), v = y.next();
        if (u != v) return u < v ? -1 : 1;
        if (x.phase == 2 && y.phase == 2) return 0;
    }
}

// Sort item. Key: the detector part of the sequence after d0 as sixteen
// 16-bit slots, most significant first, relative to the bucket (d - d0 >= 1;
// the separator and everything after it 0), plus the observables as a 64-bit
// mask -- built from the source's records when the bucket is loaded.
// "complete": every detector fits the slots (<= 16 after d0, deltas < 2^16)
// and every observable id is < 64 (always true for the codes here). Within
// one bucket, complete keys compare exactly like the canonical sequences:
// slot-wise for the detectors (a prefix has its separator 0 first), then the
// observable lists via their masks (obs_less). A bucket holding any
// incomplete key is sorted with the exact comparator over the full records.
struct Item {
    uint32_t k[8];   // sixteen 16-bit detector slots, most significant first
    uint64_t obs;    // observable mask
    double prob;     // members of a group sort by probability: the fold order
    uint32_t src;
    uint32_t ndno;   // detector ids | observable ids << 16 | complete << 31
    __device__ bool complete() const { return ndno >> 31; }
};
static_assert(sizeof(Item) == sizeof(DevPlan::ItemStub), "DevPlan::ItemStub mirrors Item");
__device__ __forceinline__ Item *items_of(const DevPlan &p) { return reinterpret_cast<Item *>(p.items); }

// Word mask of the detector bits (ids < D) of word t.
__device__ __forceinline__ uint64_t det_mask(uint32_t t, uint32_t D) {
    const uint32_t b0 = t * 64;
    return b0 + 64 <= D ? ~0ull : b0 >= D ? 0 : (1ull << (D - b0)) - 1;
}

// Item of a source with at most 4 records, all in registers: records sorted
// by word with a compare-swap network, detector ids generated in order.
__device__ __forceinline__ Item make_item_small(const DevPlan &p, uint32_t s, uint32_t n, uint32_t D) {
    uint32_t t[4];
    uint64_t w[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
        t[j] = (uint32_t)j < n ? p.rtile[rec_at(p, s, j)] : 0xFFFFFFFFu;
        w[j] = (uint32_t)j < n ? p.rbits[rec_at(p, s, j)] : 0;
    }
    auto cs = [&](int a, int b) {
        const bool sw = t[a] > t[b];
        const uint32_t ta = sw ? t[b] : t[a], tb = sw ? t[a] : t[b];
        const uint64_t wa = sw ? w[b] : w[a], wb = sw ? w[a] : w[b];
        t[a] = ta;
        t[b] = tb;
        w[a] = wa;
        w[b] = wb;
    };
    cs(0, 1);
    cs(2, 3);
    cs(0, 2);
    cs(1, 3);
    cs(1, 2);
    // Detector ids in order (records sorted by word, bits ascending): the
    // first is the bucket (q0), the next ones go to 16-bit slots relative to
    // it, four per 64-bit word, most significant first. Observables: a mask.
    uint64_t kw[4] = {0, 0, 0, 0};
    uint32_t q0 = 0, cnt = 0, nobs = 0;
    bool fits = true;
    uint64_t obs = 0;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        if (t[j] == 0xFFFFFFFFu) continue;
        const uint64_t dm = det_mask(t[j], D);
        for (uint64_t m = w[j] & dm; m; m &= m - 1) {
            const uint32_t id1 = t[j] * 64 + (uint32_t)__ffsll((long long)m);  // id + 1
            if (cnt == 0) {
                q0 = id1;
            } else {
                const uint32_t slot = cnt - 1, v = id1 - q0;
                if (slot >= 15 || v >= 0xFFFFu) fits = false;  // no room for the separator / delta too wide
                if (slot < 16) {
                    const uint64_t add = (uint64_t)(v & 0xFFFF) << (48 - 16 * (slot & 3));
                    const uint32_t wi = slot >> 2;
                    kw[0] |= wi == 0 ? add : 0;
                    kw[1] |= wi == 1 ? add : 0;
                    kw[2] |= wi == 2 ? add : 0;
                    kw[3] |= wi == 3 ? add : 0;
                }
            }
            cnt++;
        }
        for (uint64_t ob = w[j] & ~dm; ob; ob &= ob - 1) {
            const uint32_t o = t[j] * 64 + (uint32_t)__ffsll((long long)ob) - 1 - D;
            if (o < 64) obs |= 1ull << o;
            else fits = false;
            nobs++;
        }
    }
    const uint32_t ndno = cnt | nobs << 16;  // id counts (the DEM's offsets)
    Item it;
#pragma unroll
    for (int x = 0; x < 4; x++) {
        it.k[2 * x] = (uint32_t)(kw[x] >> 32);
        it.k[2 * x + 1] = (uint32_t)kw[x];
    }
    it.obs = obs;
    it.prob = p.prob[s];
    it.src = s;
    it.ndno = ndno | ((fits && !p.force_collisions) ? 1u << 31 : 0u);
    return it;
}

// Sources with more than four records (rare): the generic path, out of line
// so that the hot path keeps its registers.
__device__ __noinline__ Item make_item_large(const DevPlan &p, uint32_t s, uint32_t D, uint32_t nrec) {
    uint32_t nd = 0, no = 0;
    for (uint32_t x = 0; x < nrec; x++) {
        const uint64_t b = p.rbits[rec_at(p, s, x)], dm = det_mask(p.rtile[rec_at(p, s, x)], D);
        nd += __popcll(b & dm);
        no += __popcll(b & ~dm);
    }
    const uint32_t ndno = nd | no << 16;
    Item it;
    SeqIt q;
    q.init(p, s, D);
    const uint32_t q0 = q.next();  // first detector + 1, or 0 (no detectors): the bucket
    bool sep = q0 == 0, fits = true;
    uint32_t sl[16];
#pragma unroll
    for (int x = 0; x < 16; x++) {
        uint32_t v = 0;
        if (!sep) {
            const uint32_t e = q.next();
            if (e == 0) sep = true;  // detector separator
            else {
                v = e - q0;
                if (v >= 0xFFFFu) fits = false;
            }
        }
        sl[x] = v & 0xFFFF;
    }
    if (!sep) fits = false;  // more than 16 detectors after d0
    uint64_t obs = 0;
    if (fits) {  // remaining: observables (o + 1) then the terminator
        for (uint32_t e; (e = q.next()) != 0;) {
            if (e > 64) {
                fits = false;
                break;
            }
            obs |= 1ull << (e - 1);
        }
    }
#pragma unroll
    for (int w = 0; w < 8; w++) it.k[w] = sl[2 * w] << 16 | sl[2 * w + 1];
    it.obs = obs;
    it.prob = p.prob[s];
    it.src = s;
    it.ndno = ndno | ((fits && !p.force_collisions) ? 1u << 31 : 0u);
    return it;
}

__device__ __forceinline__ Item make_item(const DevPlan &p, uint32_t s, uint32_t D) {
    const uint32_t nrec = p.cnt[s];
    return nrec <= 4 ? make_item_small(p, s, nrec, D) : make_item_large(p, s, D, nrec);
}

// Lexicographic compare of two sorted id lists given as masks (a != b): at
// the smallest id x in exactly one list, the list holding x is smaller iff
// the other list continues past x (a list that ends there is a prefix).
__device__ __forceinline__ int obs_cmp(uint64_t a, uint64_t b) {
    if (a == b) return 0;
    const uint32_t x = (uint32_t)__ffsll((long long)(a ^ b)) - 1;
    const uint64_t above = x == 63 ? 0 : ~0ull << (x + 1);
    if ((a >> x) & 1) return (b & above) ? -1 : 1;
    return (a & above) ? 1 : -1;
}

__device__ __forceinline__ int key_cmp(const Item &a, const Item &b) {
#pragma unroll
    for (int w = 0; w < 8; w++)
        if (a.k[w] != b.k[w]) return a.k[w] < b.k[w] ? -1 : 1;
    return obs_cmp(a.obs, b.obs);
}

// Canonical compare of two items of one bucket (0: identical signatures).
// EXACT: some key of the bucket is incomplete -- compare the full records.
template <bool EXACT>
__device__ __forceinline__ int sig_cmp(const DevPlan &p, const Item &a, const Item &b, uint32_t D) {
    if (EXACT) return seq_cmp(p, a.src, b.src, D);
    return key_cmp(a, b);
}

// Sort order: signature, then ascending probability -- the order the
// reference folds a group in (dem.cpp:97-106) -- then source id.
template <bool EXACT>
__device__ __forceinline__ bool item_less(const DevPlan &p, const Item &a, const Item &b, uint32_t D) {
    const int c = sig_cmp<EXACT>(p, a, b, D);
    if (c) return c < 0;
    if (a.prob != b.prob) return a.prob < b.prob;
    return a.src < b.src;
}

// ---------------------------------------------------------------- R1 keys
// Per source with a nonempty signature (empty ones are dropped, dem.cpp:93):
// bucket (circuit, first detector) with its slot claimed by a counting-sort
// atomic (the id counts are taken when the sort item is built).
// Source loops of the reduce: each CTA takes one contiguous chunk of sources
// (threads stride by blockDim: coalesced), and each thread caches the circuit
// its sources belong to (a circuit spans thousands of sources).
struct CircCache {
    uint64_t lo = 1, hi = 0;
    uint32_t D = 0, bucket_base = 0;
    __device__ __forceinline__ void at(const DevPlan &p, uint64_t s) {
        if (s >= lo && s < hi) return;
        const uint64_t *circ_src = arr<uint64_t>(p, p.lay.circ_src);
        const uint32_t c = find_u64(circ_src, p.tot.C, s);
        lo = circ_src[c];
        hi = circ_src[c + 1];
        const CircuitMeta &m = arr<CircuitMeta>(p, p.lay.meta)[c];
        D = m.D;
        bucket_base = m.bucket_base;
    }
};

template <class F>
__device__ __forceinline__ void for_sources(const DevPlan &p, F &&f) {
    const uint64_t S = p.tot.sources;
    const uint64_t chunk = ((S + gridDim.x - 1) / gridDim.x + blockDim.x - 1) / blockDim.x * blockDim.x;
    const uint64_t s0 = (uint64_t)blockIdx.x * chunk, s1 = min(S, s0 + chunk);
    CircCache cc;
    for (uint64_t s = s0 + threadIdx.x; s < s1; s += blockDim.x) f(s, cc);
}

__global__ void key_kernel(__grid_constant__ const DevPlan p) {
    for_sources(p, [&](uint64_t s, CircCache &cc) {
        const uint32_t n = p.cnt[s];
        if (n == 0 || n > p.K) return;  // n > K: capacity re-run (record_overflow)
        cc.at(p, s);
        // The first detector lies in the lowest word (words above the one
        // holding detector D - 1 carry observables only; records are
        // nonzero): the words of every record, the bits of one.
        uint32_t tmin = 0xFFFFFFFFu, xmin = 0;
        for (uint32_t x = 0; x < n; x++) {
            const uint32_t t = p.rtile[rec_at(p, s, x)];
            if (t < tmin) {
                tmin = t;
                xmin = x;
            }
        }
        uint32_t first = 0xFFFFFFFFu;
        if (tmin * 64 < cc.D) {
            const uint64_t d = p.rbits[rec_at(p, s, xmin)] & det_mask(tmin, cc.D);
            if (d) first = tmin * 64 + (uint32_t)__ffsll((long long)d) - 1;
        }
        const uint32_t bkt = cc.bucket_base + (first == 0xFFFFFFFFu ? 0 : first + 1);
        p.s_bkt[s] = bkt;
        p.s_pos[s] = atomicAdd(&p.bcount[bkt], 1u);
    });
}

// R3: counting-sort scatter. Each source's sort item (key built from its
// records, probability, id counts) is written to its bucket slot, so the
// bucket kernel reads every bucket as one contiguous run -- random gathers
// (latency) become scattered stores (bandwidth).
__global__ void __launch_bounds__(512, 3) scatter_kernel(__grid_constant__ const DevPlan p) {
    for_sources(p, [&](uint64_t s, CircCache &cc) {
        const uint32_t n = p.cnt[s];
        if (n == 0 || n > p.K) return;
        // the slot's loads (bucket -> its offset) are issued first and land
        // while the item is built from the records
        const uint32_t bkt = p.s_bkt[s], pos = p.s_pos[s];
        const uint32_t bo = p.boff[bkt].x;
        cc.at(p, s);
        const Item it = make_item(p, (uint32_t)s, cc.D);
        const uint64_t at = (uint64_t)bo + pos;
        if (at >= p.items_cap) {  // capacity re-run with the learned count
            atomicOr(&p.hdr->items_overflow, 1u);
            return;
        }
        // 16-byte stores where the 56-byte item allows (every other slot is 16-byte aligned)
        const uint64_t *w = reinterpret_cast<const uint64_t *>(&it);
        uint64_t *d = reinterpret_cast<uint64_t *>(items_of(p) + at);
        if ((at & 1) == 0) {
            reinterpret_cast<ulonglong2 *>(d)[0] = make_ulonglong2(w[0], w[1]);
            reinterpret_cast<ulonglong2 *>(d)[1] = make_ulonglong2(w[2], w[3]);
            reinterpret_cast<ulonglong2 *>(d)[2] = make_ulonglong2(w[4], w[5]);
            d[6] = w[6];
        } else {
            d[0] = w[0];
            reinterpret_cast<ulonglong2 *>(d + 1)[0] = make_ulonglong2(w[1], w[2]);
            reinterpret_cast<ulonglong2 *>(d + 1)[1] = make_ulonglong2(w[3], w[4]);
            reinterpret_cast<ulonglong2 *>(d + 1)[2] = make_ulonglong2(w[5], w[6]);
        }
    });
}

__device__ __forceinline__ uint32_t bucket_circuit(const DevPlan &p, uint64_t b) {
    return find_u32(arr<uint32_t>(p, p.lay.circ_bkt), p.tot.C, (uint32_t)b);
}

// Group starting at sorted position i0 of a bucket (slot base; at(x) is the
// item at sorted position x): walks to the group's end, folding the members'
// probabilities -- already ascending -- from 0 (merge_prob, dem.cpp:97-106),
// and files edge g: representative source, probability, id counts (returned).
template <bool EXACT, class At>
__device__ __forceinline__ uint32_t emit_group(const DevPlan &p, uint32_t base, uint32_t g, const At &at, uint32_t i0,
                                               uint32_t n, uint32_t D) {
    double acc = merge_prob(0.0, at(i0).prob);
    uint32_t e = i0 + 1;
    while (e < n && sig_cmp<EXACT>(p, at(e - 1), at(e), D) == 0) acc = merge_prob(acc, at(e++).prob);
    const uint32_t rep = at(i0).src;
    const uint32_t ndno = at(i0).ndno & 0x7FFFFFFFu;
    p.e_src[base + g] = rep;
    p.e_item[base + g] = 0xFFFFFFFFu;  // (exact path: ids from the records)
    p.e_prob[base + g] = acc;
    p.e_ndno[base + g] = ndno;
    return ndno;
}

// Groups of a sorted bucket, one warp: start flags by chunks of 32, group
// ids by ballot prefix, one edge per group.
template <bool EXACT, class At>
__device__ __forceinline__ void groups_warp(const DevPlan &p, uint32_t b, uint32_t base, uint32_t n, uint32_t D,
                                            const At &at) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t ng = 0, nd = 0, no = 0;
    for (uint32_t c0 = 0; c0 < n; c0 += 32) {
        const uint32_t i = c0 + lane;
        const bool start = i < n && (i == 0 || sig_cmp<EXACT>(p, at(i - 1), at(i), D) != 0);
        const uint32_t starts = __ballot_sync(0xffffffffu, start);
        if (start) {
            const uint32_t v = emit_group<EXACT>(p, base, ng + __popc(starts & ((1u << lane) - 1)), at, i, n, D);
            nd += v & 0xFFFF;
            no += v >> 16;
        }
        ng += __popc(starts);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        nd += __shfl_xor_sync(0xffffffffu, nd, d);
        no += __shfl_xor_sync(0xffffffffu, no, d);
    }
    if (lane == 0) {
        p.ecount[b] = ng;
        p.eids[b] = make_uint2(nd, no);
    }
}

// Branch-free "o sorts before m" for complete keys: key words, then the
// observable lists (obs_cmp rule), then probability bits (nonnegative
// doubles order like their bits), then source id. No divergence: every
// lane of a warp compares against the same broadcast item.
__device__ __forceinline__ uint32_t item_lt(const Item &o, const Item &m) {
    bool lt = false, eq = true;
#pragma unroll
    for (int w = 0; w < 8; w++) {
        lt |= eq && o.k[w] < m.k[w];
        eq &= o.k[w] == m.k[w];
    }
    const uint64_t d = o.obs ^ m.obs;
    const uint32_t x = (uint32_t)__ffsll((long long)d) - 1;  // valid when d != 0
    const uint64_t above = x >= 63 ? 0 : ~0ull << (x + 1);
    const bool x_in_o = (o.obs >> (x & 63)) & 1;
    const bool obs_lt = d != 0 && (x_in_o ? (m.obs & above) != 0 : (o.obs & above) == 0);
    lt |= eq && obs_lt;
    eq &= d == 0;
    const uint64_t po = (uint64_t)__double_as_longlong(o.prob), pm = (uint64_t)__double_as_longlong(m.prob);
    lt |= eq && po < pm;
    eq &= po == pm;
    lt |= eq && o.src < m.src;
    return lt ? 1u : 0u;
}

// ---------------------------------------------------------------- grouping
// A bucket is grouped by a team (one warp, or one CTA for large buckets)
// with hashing instead of sorting all its sources: sources with the same
// signature are typically ten to a group (idle and same-qubit errors of
// consecutive layers), so only the groups are sorted.
//   1. shared-memory open-addressing table: each item finds its group's
//      representative by hash + FULL key compare (never a merge on a hash);
//   2. counting sort of members by representative, member probabilities
//      gathered per group, sorted ascending, folded from 0 (dem.cpp:97-106);
//   3. the groups (distinct signatures) sorted canonically by their keys;
//   4. one edge per group in that order.
// Items stay in global memory (the bucket's contiguous run; L1-resident).

__device__ __forceinline__ uint32_t item_hash(const Item &it) {
    uint64_t h = 0x9e3779b97f4a7c15ull ^ it.obs;
#pragma unroll
    for (int w = 0; w < 8; w += 2) h = mix64(h ^ ((uint64_t)it.k[w] << 32 | it.k[w + 1]));
    return (uint32_t)(h >> 32);
}

__device__ __forceinline__ bool key_eq(const Item &a, const Item &b) {
    bool eq = a.obs == b.obs;
#pragma unroll
    for (int w = 0; w < 8; w++) eq &= a.k[w] == b.k[w];
    return eq;
}

struct WarpTeam {
    __device__ uint32_t t0() const { return threadIdx.x & 31; }
    __device__ uint32_t nt() const { return 32; }
    __device__ void sync() const { __syncwarp(); }
    __device__ bool any(bool v) const { return __any_sync(0xffffffffu, v); }
};
struct CtaTeam {
    __device__ uint32_t t0() const { return threadIdx.x; }
    __device__ uint32_t nt() const { return blockDim.x; }
    __device__ void sync() const { __syncthreads(); }
    __device__ bool any(bool v) const { return __syncthreads_or(v) != 0; }
};

// Shared workspace of one team for a bucket of up to `cap` (< 65535) items;
// 16-bit item indices keep a warp's workspace at 5.6 KB (occupancy).
struct GroupWs {
    double *mp;      // [cap] member probabilities grouped; [off[r]] = folded probability
    uint32_t *cnt;   // [cap] members per representative, then fill counters
    uint32_t *tot;   // [4] team scratch: group count, id sums
    uint16_t *tab;   // [tcap] representative item or 0xFFFF
    uint16_t *rep;   // [cap] item -> representative
    uint16_t *off;   // [cap] member offset per representative
    uint16_t *grp;   // [cap] representatives (groups), canonical order after the sort
    uint32_t tcap;   // power of two >= 2 cap
    __device__ static size_t bytes(uint32_t cap, uint32_t tcap) {
        return ((size_t)cap * (8 + 4 + 2 * 3) + 16 + (size_t)tcap * 2 + 15) & ~(size_t)15;
    }
    __device__ void carve(uint8_t *base, uint32_t cap, uint32_t tc) {
        tcap = tc;
        mp = reinterpret_cast<double *>(base);  // 8-byte aligned first
        cnt = reinterpret_cast<uint32_t *>(mp + cap);
        tot = cnt + cap;
        tab = reinterpret_cast<uint16_t *>(tot + 4);
        rep = tab + tcap;
        off = rep + cap;
        grp = off + cap;
    }
};

// Exclusive prefix of cnt[0..n) into off[], listing representatives (cnt > 0)
// in grp[] (ascending item order); returns the group count. Team-wide.
template <class Team>
__device__ __forceinline__ uint32_t scan_groups(const Team &tm, const GroupWs &w, uint32_t n) {
    const uint32_t t0 = tm.t0(), nt = tm.nt();
    const uint32_t per = (n + nt - 1) / nt, a = min(n, t0 * per), e = min(n, a + per);
    uint32_t sm = 0, sg = 0;
    for (uint32_t i = a; i < e; i++) {
        sm += w.cnt[i];
        sg += w.cnt[i] != 0;
    }
    // team exclusive scan of (sm, sg): warp shuffles, then warp totals
    const uint32_t lane = threadIdx.x & 31, wid = t0 >> 5;
    uint32_t im = sm, ig = sg;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, im, d), y = __shfl_up_sync(0xffffffffu, ig, d);
        if (lane >= (uint32_t)d) {
            im += x;
            ig += y;
        }
    }
    __shared__ uint32_t s_wm[33], s_wg[33];
    uint32_t bm = 0, bg = 0;
    if (nt > 32) {
        if (lane == 31) {
            s_wm[wid] = im;
            s_wg[wid] = ig;
        }
        tm.sync();
        for (uint32_t x = 0; x < wid; x++) {
            bm += s_wm[x];
            bg += s_wg[x];
        }
    }
    uint32_t om = bm + im - sm, og = bg + ig - sg;
    for (uint32_t i = a; i < e; i++) {
        w.off[i] = (uint16_t)om;
        om += w.cnt[i];
        if (w.cnt[i]) w.grp[og++] = (uint16_t)i;
    }
    if (t0 == nt - 1) w.tot[0] = og;  // the last thread ends at the total
    tm.sync();
    const uint32_t G = w.tot[0];
    tm.sync();
    return G;
}

// Returns false, having written nothing, when some key of the bucket is
// incomplete (found while hashing): the caller takes the exact path.
template <class Team>
__device__ bool group_bucket(const DevPlan &p, const Team &tm, uint32_t b, uint32_t base, uint32_t n,
                             const Item *it, GroupWs &w) {
    const uint32_t t0 = tm.t0(), nt = tm.nt();
    for (uint32_t x = t0; x < w.tcap; x += nt) w.tab[x] = 0xFFFF;
    for (uint32_t x = t0; x < n; x += nt) w.cnt[x] = 0;
    tm.sync();
    // 1. representatives: hash + full key compare
    bool inc = false;
    for (uint32_t i = t0; i < n; i += nt) {
        const Item me = it[i];
        inc |= !me.complete();
        uint32_t h = item_hash(me) & (w.tcap - 1), r = i;
        while (true) {
            uint32_t cur = w.tab[h];
            if (cur == 0xFFFF) {
                cur = atomicCAS(&w.tab[h], (unsigned short)0xFFFF, (unsigned short)i);
                if (cur == 0xFFFF) break;  // this item founds the group
            }
            if (key_eq(it[cur], me)) {
                r = cur;
                break;
            }
            h = (h + 1) & (w.tcap - 1);
        }
        w.rep[i] = (uint16_t)r;
        atomicAdd(&w.cnt[r], 1u);
    }
    tm.sync();
    if (tm.any(inc)) return false;
    // 2. members grouped by representative; sorted ascending fold per group
    const uint32_t G = scan_groups(tm, w, n);
    constexpr bool kWarp = std::is_same<Team, WarpTeam>::value;
    {
    for (uint32_t i = t0; i < n; i += nt) {
        const uint32_t r = w.rep[i];
        w.mp[w.off[r] + atomicSub(&w.cnt[r], 1u) - 1] = it[i].prob;
    }
    tm.sync();
    for (uint32_t g = t0; g < G; g += nt) {
        const uint32_t r = w.grp[g];
        const uint32_t o = w.off[r], e = g + 1 < G ? w.off[w.grp[g + 1]] : n;
        double *v = w.mp + o;
        for (uint32_t a = o + 1; a < e; a++) {  // insertion sort of the group's probabilities
            const double x = w.mp[a];
            uint32_t z = a;
            while (z > o && w.mp[z - 1] > x) {
                w.mp[z] = w.mp[z - 1];
                z--;
            }
            w.mp[z] = x;
        }
        double acc = 0;
        for (uint32_t a = o; a < e; a++) acc = merge_prob(acc, w.mp[a]);
        v[0] = acc;
    }
    tm.sync();
    }
    // 3. groups in canonical order. A warp with at most 32 groups ranks them
    // (one group per lane, keys distinct); otherwise bitonic ("flip" form).
    if (kWarp && G <= 32) {
        const uint32_t lane = t0;
        const uint32_t mine = lane < G ? w.grp[lane] : 0;
        uint32_t rank = 0;
        Item me{};
        if (lane < G) me = it[mine];
        for (uint32_t h = 0; h < G; h++) {  // the others' keys by shuffle (all lanes take part)
            Item o;
#pragma unroll
            for (int x = 0; x < 8; x++) o.k[x] = __shfl_sync(0xffffffffu, me.k[x], h);
            o.obs = __shfl_sync(0xffffffffu, me.obs, h);
            rank += (lane < G && h != lane && key_cmp(o, me) < 0) ? 1u : 0u;
        }
        __syncwarp();
        if (lane < G) w.grp[rank] = (uint16_t)mine;
        __syncwarp();
    } else {
    uint32_t np = 1;
    while (np < G) np <<= 1;
    auto cas = [&](uint32_t x, uint32_t y) {
        const uint32_t u = w.grp[x], v = w.grp[y];
        if (key_cmp(it[v], it[u]) < 0) {
            w.grp[x] = (uint16_t)v;
            w.grp[y] = (uint16_t)u;
        }
    };
    for (uint32_t k = 2; k <= np; k <<= 1) {
        for (uint32_t x = t0; x < G; x += nt) {
            const uint32_t y = x ^ (k - 1);
            if (y > x && y < G) cas(x, y);
        }
        tm.sync();
        for (uint32_t j = k >> 2; j > 0; j >>= 1) {
            for (uint32_t x = t0; x < G; x += nt) {
                const uint32_t y = x ^ j;
                if (y > x && y < G) cas(x, y);
            }
            tm.sync();
        }
    }
    }
    // 4. edges
    uint32_t nd = 0, no = 0;
    for (uint32_t g = t0; g < G; g += nt) {
        const uint32_t r = w.grp[g];
        const uint32_t v = it[r].ndno & 0x7FFFFFFFu;
        p.e_src[base + g] = it[r].src;
        p.e_item[base + g] = base + r;  // complete key: write_kernel decodes the ids from the item
        p.e_prob[base + g] = w.mp[w.off[r]];
        p.e_ndno[base + g] = v;
        nd += v & 0xFFFF;
        no += v >> 16;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        nd += __shfl_xor_sync(0xffffffffu, nd, d);
        no += __shfl_xor_sync(0xffffffffu, no, d);
    }
    if (t0 == 0) w.tot[1] = w.tot[2] = 0;
    tm.sync();
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&w.tot[1], nd);
        atomicAdd(&w.tot[2], no);
    }
    tm.sync();
    if (t0 == 0) {
        p.ecount[b] = G;
        p.eids[b] = make_uint2(w.tot[1], w.tot[2]);
    }
    tm.sync();
    return true;
}

// Exact fallback for a bucket holding an incomplete key (pathological
// weights): rank every item with the exact comparator, then groups in order.
__device__ void bucket_exact_warp(const DevPlan &p, uint32_t b, uint32_t base, uint32_t n, uint32_t D,
                                  uint16_t *order) {
    const uint32_t lane = threadIdx.x & 31;
    const Item *it = items_of(p) + base;
    for (uint32_t i = lane; i < n; i += 32) {
        const Item m = it[i];
        uint32_t rank = 0;
        for (uint32_t j = 0; j < n; j++) rank += (j != i && item_less<true>(p, it[j], m, D)) ? 1 : 0;
        order[rank] = (uint16_t)i;
    }
    __syncwarp();
    auto at = [&](uint32_t x) -> const Item & { return it[order[x]]; };
    groups_warp<true>(p, b, base, n, D, at);
    __syncwarp();
}

// Bitonic network in its "flip" form: every comparator puts the smaller item
// first, so indices >= n act as +infinity and are skipped (no padding).
// `sync` is __syncwarp for one warp, __syncthreads for a CTA.
template <bool EXACT, class Sync>
__device__ __forceinline__ void bitonic(const DevPlan &p, Item *it, uint32_t n, uint32_t D, uint32_t t0,
                                        uint32_t nt, Sync sync) {
    uint32_t np = 1;
    while (np < n) np <<= 1;
    auto cas = [&](uint32_t i, uint32_t l) {
        const Item a = it[i], c = it[l];
        if (item_less<EXACT>(p, c, a, D)) {
            it[i] = c;
            it[l] = a;
        }
    };
    for (uint32_t k = 2; k <= np; k <<= 1) {
        for (uint32_t i = t0; i < n; i += nt) {
            const uint32_t l = i ^ (k - 1);
            if (l > i && l < n) cas(i, l);
        }
        sync();
        for (uint32_t j = k >> 2; j > 0; j >>= 1) {
            for (uint32_t i = t0; i < n; i += nt) {
                const uint32_t l = i ^ j;
                if (l > i && l < n) cas(i, l);
            }
            sync();
        }
    }
}

// One CTA, larger buckets (huge_kernel): bitonic sort, then groups.
template <bool EXACT>
__device__ void groups_cta(const DevPlan &p, uint32_t b, uint32_t base, uint32_t n, uint32_t D, const Item *it) {
    __shared__ uint32_t s_cnt[33], s_ids[2];
    if (threadIdx.x == 0) s_ids[0] = s_ids[1] = 0;
    uint32_t total = 0;
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint32_t c0 = 0; c0 < n; c0 += blockDim.x) {
        const uint32_t i = c0 + threadIdx.x;
        const bool start = i < n && (i == 0 || sig_cmp<EXACT>(p, it[i - 1], it[i], D) != 0);
        const uint32_t bal = __ballot_sync(0xffffffffu, start);
        if (lane == 0) s_cnt[w] = __popc(bal);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t run = 0;
            for (uint32_t x = 0; x < blockDim.x / 32; x++) {
                const uint32_t v = s_cnt[x];
                s_cnt[x] = run;
                run += v;
            }
            s_cnt[32] = run;
        }
        __syncthreads();
        if (start) {
            auto at = [&](uint32_t x) -> const Item & { return it[x]; };
            const uint32_t v =
                emit_group<EXACT>(p, base, total + s_cnt[w] + __popc(bal & ((1u << lane) - 1)), at, i, n, D);
            atomicAdd(&s_ids[0], v & 0xFFFF);
            atomicAdd(&s_ids[1], v >> 16);
        }
        total += s_cnt[32];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        p.ecount[b] = total;
        p.eids[b] = make_uint2(s_ids[0], s_ids[1]);
    }
    __syncthreads();
}

__device__ void bucket_cta(const DevPlan &p, uint32_t b, uint32_t n, uint32_t D, Item *it) {
    const uint32_t base = p.boff[b].x;
    __shared__ uint32_t s_inc;
    if (threadIdx.x == 0) s_inc = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
        if (!it[i].complete()) s_inc = 1;
    __syncthreads();
    if (s_inc) {
        bitonic<true>(p, it, n, D, threadIdx.x, blockDim.x, [] { __syncthreads(); });
        groups_cta<true>(p, b, base, n, D, it);
    } else {
        bitonic<false>(p, it, n, D, threadIdx.x, blockDim.x, [] { __syncthreads(); });
        groups_cta<false>(p, b, base, n, D, it);
    }
}

constexpr uint32_t kWarpTab = 512;                                   // >= 2 kWarpItems
constexpr uint32_t kWarpWs = (256 * 18 + 16 + 512 * 2 + 15) & ~15u;  // GroupWs::bytes(256, 512)
constexpr uint32_t kHugeSmem = 196 * 1024;                            // huge_kernel dynamic smem

// One warp per bucket, no CTA synchronisation: empty buckets, buckets of up
// to kWarpItems sources (group_bucket in the warp's workspace, or the exact
// fallback); larger ones are listed for huge_kernel.
__global__ void __launch_bounds__(kBucketThreads) bucket_kernel(__grid_constant__ const DevPlan p) {
    __shared__ __align__(16) uint8_t ws[(kBucketThreads / 32) * kWarpWs];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    GroupWs w;
    w.carve(ws + warp * kWarpWs, kWarpItems, kWarpTab);
    const uint64_t NB = p.tot.buckets;
    const CircuitMeta *meta = arr<CircuitMeta>(p, p.lay.meta);
    const uint64_t warps = (uint64_t)gridDim.x * (kBucketThreads / 32);
    if (p.hdr->items_overflow) return;  // re-run with a larger item array
    for (uint64_t b = ((uint64_t)blockIdx.x * kBucketThreads + threadIdx.x) >> 5; b < NB; b += warps) {
        const uint32_t base = p.boff[b].x, n = p.boff[b + 1].x - base;
        if (n == 0) {
            if (lane == 0) {
                p.ecount[b] = 0;
                p.eids[b] = make_uint2(0, 0);
            }
            continue;
        }
        if (n > kWarpItems) {
            if (lane == 0) p.huge[atomicAdd(&p.hdr->huge_count, 1u)] = (uint32_t)b;
            continue;
        }
        const Item *it = items_of(p) + base;
        if (!group_bucket(p, WarpTeam{}, (uint32_t)b, base, n, it, w))  // (an incomplete key: exact ranks)
            bucket_exact_warp(p, (uint32_t)b, base, n, meta[bucket_circuit(p, b)].D,
                              reinterpret_cast<uint16_t *>(w.tab));
    }
}

// Buckets too large for a warp: one CTA each, group_bucket in up to 196 KB
// of dynamic shared memory; the exact CTA sort (in place in the bucket's own
// run of the item array) for incomplete keys or buckets beyond that.
__global__ void __launch_bounds__(256) huge_kernel(__grid_constant__ const DevPlan p) {
    extern __shared__ __align__(16) uint8_t hsm[];
    if (p.hdr->items_overflow) return;
    const uint32_t nh = p.hdr->huge_count;
    const CircuitMeta *meta = arr<CircuitMeta>(p, p.lay.meta);
    __shared__ uint32_t s_inc;
    for (uint32_t i = blockIdx.x; i < nh; i += gridDim.x) {
        const uint32_t b = p.huge[i];
        const uint32_t base = p.boff[b].x, n = p.boff[b + 1].x - base;
        Item *it = items_of(p) + base;
        if (threadIdx.x == 0) s_inc = 0;
        __syncthreads();
        for (uint32_t x = threadIdx.x; x < n; x += blockDim.x)
            if (!it[x].complete()) s_inc = 1;
        __syncthreads();
        uint32_t tc = 1;
        while (tc < 2 * n) tc <<= 1;
        if (!s_inc && GroupWs::bytes(n, tc) <= kHugeSmem) {
            GroupWs w;
            w.carve(hsm, n, tc);
            group_bucket(p, CtaTeam{}, b, base, n, it, w);
        } else {
            bucket_cta(p, b, n, meta[bucket_circuit(p, b)].D, it);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- R6 output
// Bucket b's groups become edges [eoff, eoff + ecount) of the flat DEM, ids
// expanded from the representative's records in word order (bit b < D ->
// detector b, else observable b - D; dem.cpp:108-116).
__global__ void write_kernel(__grid_constant__ const DevPlan p, const uint4 *out_total) {
    const uint64_t NB = p.tot.buckets;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const CircuitMeta *meta = arr<CircuitMeta>(p, p.lay.meta);
    const uint4 tot = *out_total;
    const uint64_t bE = p.base_in[0], bD = p.base_in[1], bO = p.base_in[2];
    const bool fits = (uint64_t)tot.y <= p.ids_cap && (uint64_t)tot.z <= p.ids_cap && (uint64_t)tot.x <= p.e_cap;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        DeviceHeader h = *p.hdr;
        if (!fits) {
            h.num_det_ids = 0xFFFFFFFFu;  // capacity overflow marker: re-run larger
        } else {
            h.num_edges = tot.x;
            h.num_det_ids = tot.y;
            h.num_obs_ids = tot.z;
            p.o_det_off[tot.x] = bD + tot.y;
            p.o_obs_off[tot.x] = bO + tot.z;
        }
        *p.hdr = h;
        *p.hdr_out = h;
        p.base_out[0] = bE + tot.x;
        p.base_out[1] = bD + tot.y;
        p.base_out[2] = bO + tot.z;
        p.base_out[3] = p.base_in[3] + p.tot.C;
    }
    if (!fits || p.hdr->items_overflow) return;
    {  // per-circuit edge offsets (the bucket scan at each circuit's first bucket)
        const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
        if (t <= p.tot.C) p.o_edge_off[t] = bE + (t < p.tot.C ? p.oscan[meta[t].bucket_base].x : tot.x);
    }
    for (uint64_t b = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < NB; b += warps) {
        const uint32_t ne = p.ecount[b];
        if (ne == 0) continue;
        const uint4 o = p.oscan[b];  // (edges, det ids, obs ids) before this bucket
        const uint32_t base = p.boff[b].x;
        const CircuitMeta &cm = meta[bucket_circuit(p, b)];
        const uint32_t D = cm.D, q0 = (uint32_t)b - cm.bucket_base;  // first detector + 1 (0: none)
        const Item *items = items_of(p);
        uint32_t dcar = 0, ocar = 0;
        for (uint32_t k0 = 0; k0 < ne; k0 += 32) {
            const uint32_t k = k0 + lane;
            uint32_t nd = 0, no = 0;
            if (k < ne) {
                const uint32_t v = p.e_ndno[base + k];
                nd = v & 0xFFFF;
                no = v >> 16;
            }
            uint32_t di = nd, oi = no;  // inclusive warp scans
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t a = __shfl_up_sync(0xffffffffu, di, d), c = __shfl_up_sync(0xffffffffu, oi, d);
                if (lane >= (uint32_t)d) {
                    di += a;
                    oi += c;
                }
            }
            if (k < ne) {
                const uint64_t e = (uint64_t)o.x + k;
                const uint32_t d0 = o.y + dcar + di - nd, o0 = o.z + ocar + oi - no;
                p.o_det_off[e] = bD + d0;
                p.o_obs_off[e] = bO + o0;
                p.o_prob[e] = p.e_prob[base + k];
                const uint32_t ii = p.e_item[base + k];
                if (ii != 0xFFFFFFFFu) {  // complete key: detectors q0 - 1 + slot deltas, observables by mask
                    const Item q = items[ii];
                    uint32_t wd = d0, wo = o0;
                    if (q0) {
                        p.o_det[wd++] = q0 - 1;
                        for (uint32_t x = 0; x < 16; x++) {
                            const uint32_t v = (q.k[x >> 1] >> ((x & 1) ? 0 : 16)) & 0xFFFF;
                            if (v == 0) break;
                            p.o_det[wd++] = q0 - 1 + v;
                        }
                    }
                    for (uint64_t ob = q.obs; ob; ob &= ob - 1) p.o_obs[wo++] = (uint32_t)__ffsll((long long)ob) - 1;
                } else {  // ids from the representative's records, in word order
                    const uint32_t r = p.e_src[base + k];
                    uint8_t ord[16];
                    const uint32_t n = min(p.cnt[r], 16u);
                    sig_order(p, r, n, ord);
                    uint32_t wd = d0, wo = o0;
                    for (uint32_t x = 0; x < n; x++) {
                        const uint32_t t = p.rtile[rec_at(p, r, ord[x])];
                        uint64_t bits = p.rbits[rec_at(p, r, ord[x])];
                        while (bits) {
                            const uint32_t id = t * 64 + (uint32_t)__ffsll((long long)bits) - 1;
                            bits &= bits - 1;
                            if (id < D) p.o_det[wd++] = id;
                            else p.o_obs[wo++] = id - D;
                        }
                    }
                }
            }
            dcar += __shfl_sync(0xffffffffu, di, 31);
            ocar += __shfl_sync(0xffffffffu, oi, 31);
        }
    }
}

// Mapped output: the output region and the header into mapped pinned host
// memory (coalesced stores over PCIe; sizes from the device header).
__global__ void copy_out_kernel(__grid_constant__ const DevPlan p) {
    const DeviceHeader hd = *p.hdr;
    const bool ok = hd.num_det_ids != 0xFFFFFFFFu && !hd.items_overflow && !hd.record_overflow && !hd.pool_overflow;
    const uint64_t E = hd.num_edges, nd = ok ? hd.num_det_ids : 0, no = hd.num_obs_ids, C = p.tot.C;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x, t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (ok) {
        for (uint64_t i = t0; i <= E; i += stride) {
            p.hmap.det_off[i] = p.o_det_off[i];
            p.hmap.obs_off[i] = p.o_obs_off[i];
            if (i < E) p.hmap.probs[i] = p.o_prob[i];
        }
        for (uint64_t i = t0; i < nd; i += stride) p.hmap.det_ids[i] = p.o_det[i];
        for (uint64_t i = t0; i < no; i += stride) p.hmap.obs_ids[i] = p.o_obs[i];
        for (uint64_t i = t0; i <= C; i += stride) p.hmap.edge_off[i] = p.o_edge_off[i];
    }
    if (t0 == 0) *p.hmap.hdr = hd;
}

}  // namespace red

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
// sequences. seq[0] picks the bucket. Within a bucket (d0 equal), the
// detector part compares like the CONSECUTIVE differences d1-d0, d2-d1, ...
// (each >= 1; a list that ends scores 0, so a prefix sorts first): equal
// prefixes of ids are equal prefixes of differences. Those differences,
// 12 bits each, ten of them, are the 128-bit sort key of a 32-byte sort item;
// the observables follow as a 64-bit mask (obs_cmp). A signature that does not
// fit (more than 11 detectors, a difference over 4095, an observable id over
// 63) keeps its source id instead and its bucket is compared exactly over the
// full records, so distinct signatures never merge (dem.cpp:73-78,
// test_dem.cpp:94-101).

#include <type_traits>

namespace red {

constexpr uint32_t kBucketThreads = 128, kWarpItems = 256;  // bucket_kernel: a warp groups up to kWarpItems


// Records per source the exact paths handle (signatures spanning up to this
// many nonzero 64-bit words; the host grows the record slots up to it).
constexpr uint32_t kMaxRecords = 64;

// Slots of source s's records sorted by word (insertion sort, n <= kMaxRecords).
__device__ __forceinline__ uint32_t sig_order(const DevPlan &p, uint64_t s, uint32_t n, uint8_t *ord) {
    uint32_t tile[kMaxRecords];
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
    uint8_t ord[kMaxRecords];

    __device__ void init(const DevPlan &pl, uint64_t src, uint32_t d) {
        rtile = pl.rtile + src;
        rbits = pl.rbits + src;
        stride = pl.tot.sources;
        D = d;
        n = min(pl.cnt[src], kMaxRecords);
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

// Sort item (32 bytes, two 16-byte stores / loads).
//   k0: differences 1..5, k1: differences 6..10 -- 12 bits each, most
//       significant first (bits 63..52 hold the first), 0 after the last;
//       k1 bit 0: INCOMPLETE (the key did not fit; obs then holds the source)
//       k1 bit 1: the signature has detectors (the bucket's q0 != 0; equal
//       for every item of a bucket, so it never changes an order)
//   obs: observable mask (complete items)
//   prob: the source's probability (members of a group fold in its order)
// No source id: complete items decode their ids from the key (write_kernel),
// and order ties inside a bucket break by position.
struct Item {
    uint64_t k0, k1, obs;
    double prob;
    __device__ bool complete() const { return !(k1 & 1); }
    __device__ uint32_t src() const { return (uint32_t)obs; }
};
static_assert(sizeof(Item) == sizeof(DevPlan::ItemStub), "DevPlan::ItemStub mirrors Item");
__device__ __forceinline__ Item *items_of(const DevPlan &p) { return reinterpret_cast<Item *>(p.items); }

constexpr uint32_t kKeyFields = 10, kKeyDeltaMax = 4095;

__device__ __forceinline__ void key_put(uint64_t &k0, uint64_t &k1, uint32_t f, uint64_t v) {
    const uint32_t sh = 52 - 12 * (f % 5);
    if (f < 5) k0 |= v << sh;
    else k1 |= v << sh;
}

__device__ __forceinline__ uint32_t key_get(const Item &it, uint32_t f) {
    return (uint32_t)(((f < 5 ? it.k0 : it.k1) >> (52 - 12 * (f % 5))) & 0xFFF);
}

// Detectors after d0 in a complete key. Its nonzero fields form a prefix, so
// the lowest set field bit names the last one (field f of a word spans bits
// 52 - 12 f .. 63 - 12 f; k1's bits 0..3 are flags).
__device__ __forceinline__ uint32_t key_len(const Item &it) {
    const uint64_t h = it.k1 & ~15ull;
    if (h) return 5 + (63 - (uint32_t)(__ffsll((long long)h) - 1)) / 12 + 1;
    if (it.k0) return (63 - (uint32_t)(__ffsll((long long)it.k0) - 1)) / 12 + 1;
    return 0;
}

constexpr uint64_t kItemIncomplete = 1, kItemHasDet = 2;

__device__ __forceinline__ Item incomplete_item(uint32_t s, double prob) {
    Item it;
    it.k0 = 0;
    it.k1 = kItemIncomplete;
    it.obs = s;
    it.prob = prob;
    return it;
}

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
    // first is the bucket, the next ones go to the key as differences.
    uint64_t k0 = 0, k1 = 0, obs = 0;
    uint32_t prev = 0, cnt = 0;
    bool fits = true;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        if (t[j] == 0xFFFFFFFFu) continue;
        const uint64_t dm = det_mask(t[j], D);
        for (uint64_t m = w[j] & dm; m; m &= m - 1) {
            const uint32_t id = t[j] * 64 + (uint32_t)__ffsll((long long)m) - 1;
            if (cnt) {
                const uint32_t dv = id - prev;
                if (cnt > kKeyFields || dv > kKeyDeltaMax) fits = false;
                else key_put(k0, k1, cnt - 1, dv);
            }
            prev = id;
            cnt++;
        }
        for (uint64_t ob = w[j] & ~dm; ob; ob &= ob - 1) {
            const uint32_t o = t[j] * 64 + (uint32_t)__ffsll((long long)ob) - 1 - D;
            if (o < 64) obs |= 1ull << o;
            else fits = false;
        }
    }
    const double prob = p.prob[s];
    if (!fits || p.force_collisions) return incomplete_item(s, prob);
    Item it;
    it.k0 = k0;
    it.k1 = k1 | (cnt ? kItemHasDet : 0);
    it.obs = obs;
    it.prob = prob;
    return it;
}

// Sources with more than four records (rare): the generic path, out of line
// so that the hot path keeps its registers.
__device__ __noinline__ Item make_item_large(const DevPlan &p, uint32_t s, uint32_t D) {
    SeqIt q;
    q.init(p, s, D);
    uint32_t prev = q.next();  // first detector + 1, or 0 (no detectors): the bucket
    const bool has_det = prev != 0;
    bool sep = prev == 0, fits = true;
    uint64_t k0 = 0, k1 = 0, obs = 0;
    for (uint32_t f = 0; !sep; f++) {
        const uint32_t e = q.next();
        if (e == 0) {
            sep = true;  // detector separator
        } else {
            if (f >= kKeyFields || e - prev > kKeyDeltaMax) fits = false;
            else key_put(k0, k1, f, e - prev);
            prev = e;
        }
    }
    for (uint32_t e; (e = q.next()) != 0;) {  // observables (o + 1), then the terminator
        if (e > 64) fits = false;
        else obs |= 1ull << (e - 1);
    }
    const double prob = p.prob[s];
    if (!fits || p.force_collisions) return incomplete_item(s, prob);
    Item it;
    it.k0 = k0;
    it.k1 = k1 | (has_det ? kItemHasDet : 0);
    it.obs = obs;
    it.prob = prob;
    return it;
}

__device__ __forceinline__ Item make_item(const DevPlan &p, uint32_t s, uint32_t D) {
    const uint32_t nrec = p.cnt[s];
    return nrec <= 4 ? make_item_small(p, s, nrec, D) : make_item_large(p, s, D);
}

// Item of a signature held in registers (fused items: the direct traversal
// owns all TM words of its circuit, word w = ids [64 w, 64 w + 64)). Ids come
// out ascending, word by word, bit by bit; each detector id pushes its
// difference into a 128-bit shift register (branch-free: the first id's
// "difference" is pushed too and shifted out at the end), observables are
// shifted into their mask a word at a time. *local = the circuit-local bucket
// (first detector + 1, or 0 without detectors).
template <int TM>
__device__ __forceinline__ Item item_of_words(const uint64_t (&v)[TM], uint32_t tw, uint32_t D, double prob,
                                              uint32_t src, bool force, uint32_t *local) {
    uint64_t hi = 0, lo = 0, obs = 0;
    uint32_t prev = 0, cnt = 0, first = 0;
    bool fits = true;
    const uint32_t wD = D >> 6;
    const uint64_t lowD = (1ull << (D & 63)) - 1;
#pragma unroll
    for (int w = 0; w < TM; w++) {
        if ((uint32_t)w >= tw || !v[w]) continue;
        const uint64_t dm = (uint32_t)w < wD ? ~0ull : (uint32_t)w == wD ? lowD : 0ull;
        for (uint64_t m = v[w] & dm; m; m &= m - 1) {
            const uint32_t id = (uint32_t)w * 64 + (uint32_t)__ffsll((long long)m) - 1;
            const uint32_t dv = id - prev;
            fits &= dv <= kKeyDeltaMax || cnt == 0;
            first = cnt == 0 ? id : first;
            hi = hi << 12 | lo >> 52;
            lo = lo << 12 | dv;
            prev = id;
            cnt++;
        }
        const uint64_t ob = v[w] & ~dm;  // observable o = 64 w + bit - D
        if (ob) {
            const int sh = w * 64 - (int)D;
            if (sh >= 64) fits = false;
            else if (sh >= 0) {
                if (sh > 0 && (ob >> (64 - sh))) fits = false;
                obs |= ob << sh;
            } else {
                obs |= ob >> -sh;
            }
        }
    }
    *local = cnt ? first + 1 : 0;
    if (cnt > kKeyFields + 1 || !fits || force) return incomplete_item(src, prob);
    // n = cnt - 1 differences in the low 12 n bits: align field 0 at bit 119
    // (k0 = bits 119..60 << 4, k1 = bits 59..0 << 4, as key_put lays them out)
    uint64_t k0 = 0, k1 = 0;
    if (cnt > 1) {
        const uint32_t s = 12 * (kKeyFields + 1 - cnt);
        if (s >= 64) {
            hi = lo << (s - 64);
            lo = 0;
        } else if (s > 0) {
            hi = hi << s | lo >> (64 - s);
            lo <<= s;
        }
        k0 = (hi << 4 | lo >> 60) << 4;
        k1 = lo << 4;
    }
    Item it;
    it.k0 = k0;
    it.k1 = k1 | (cnt ? kItemHasDet : 0);
    it.obs = obs;
    it.prob = prob;
    return it;
}

__device__ __forceinline__ void store_item(Item *dst, const Item &it) {
    ulonglong2 *d = reinterpret_cast<ulonglong2 *>(dst);
    d[0] = make_ulonglong2(it.k0, it.k1);
    d[1] = make_ulonglong2(it.obs, (unsigned long long)__double_as_longlong(it.prob));
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
    if (a.k0 != b.k0) return a.k0 < b.k0 ? -1 : 1;
    if (a.k1 != b.k1) return a.k1 < b.k1 ? -1 : 1;
    return obs_cmp(a.obs, b.obs);
}

// The bucket an item is compared in: D of its circuit and q0 = first
// detector + 1 (0: a bucket of observable-only signatures).
struct BucketCtx {
    uint32_t D, q0;
};

// Lazy canonical sequence of one item: decoded from a complete key, or
// generated from the source's records (SeqIt) for an incomplete one.
struct ItemSeq {
    SeqIt r;
    uint64_t k0, k1, obs;
    uint32_t f, prev, state;  // state 0: d0, 1: differences, 2: observables, 3: done
    bool rec;
    __device__ void init(const DevPlan &p, const Item &it, BucketCtx c) {
        rec = !it.complete();
        if (rec) {
            r.init(p, it.src(), c.D);
            return;
        }
        k0 = it.k0;
        k1 = it.k1;
        obs = it.obs;
        f = 0;
        prev = c.q0;
        state = 0;
    }
    __device__ bool done() const { return rec ? r.phase == 2 : state == 3; }
    __device__ uint32_t next() {
        if (rec) return r.next();
        switch (state) {
            case 0:
                state = prev ? 1 : 2;  // no detectors: the separator comes first
                return prev;
            case 1: {
                const uint32_t dv = f < kKeyFields ? key_get(Item{k0, k1, 0, 0}, f) : 0;
                f++;
                if (dv == 0) {
                    state = 2;
                    return 0;
                }
                prev += dv;
                return prev;
            }
            case 2:
                if (obs) {
                    const uint32_t x = (uint32_t)__ffsll((long long)obs);
                    obs &= obs - 1;
                    return x;
                }
                state = 3;
                return 0;
            default:
                return 0;
        }
    }
};

// Exact canonical compare of two items of one bucket (-1, 0, 1).
__device__ __forceinline__ int seq_cmp(const DevPlan &p, const Item &a, const Item &b, BucketCtx c) {
    ItemSeq x, y;
    x.init(p, a, c);
    y.init(p, b, c);
    while (true) {
        const uint32_t u = x.next(), v = y.next();
        if (u != v) return u < v ? -1 : 1;
        if (x.done() && y.done()) return 0;
    }
}

// Canonical compare of two items of one bucket (0: identical signatures).
// EXACT: some key of the bucket is incomplete -- compare the sequences.
template <bool EXACT>
__device__ __forceinline__ int sig_cmp(const DevPlan &p, const Item &a, const Item &b, BucketCtx c) {
    if (EXACT) return seq_cmp(p, a, b, c);
    return key_cmp(a, b);
}

// Sort order: signature, then ascending probability -- the order the
// reference folds a group in (dem.cpp:97-106) -- then position (ia, ib).
template <bool EXACT>
__device__ __forceinline__ bool item_less(const DevPlan &p, const Item &a, uint32_t ia, const Item &b, uint32_t ib,
                                          BucketCtx c) {
    const int s = sig_cmp<EXACT>(p, a, b, c);
    if (s) return s < 0;
    if (a.prob != b.prob) return a.prob < b.prob;
    return ia < ib;
}

// Id counts (detectors | observables << 16) of a complete key.
__device__ __forceinline__ uint32_t key_ndno(const Item &it) {
    return ((uint32_t)(it.k1 >> 1 & 1) + key_len(it)) | (uint32_t)__popcll(it.obs) << 16;
}

// Id counts of any item's signature (an incomplete one: from its records).
__device__ __forceinline__ uint32_t item_ndno(const DevPlan &p, const Item &it, BucketCtx c) {
    if (it.complete()) return key_ndno(it);
    const uint32_t s = it.src(), n = min(p.cnt[s], kMaxRecords);
    uint32_t nd = 0, no = 0;
    for (uint32_t x = 0; x < n; x++) {
        const uint64_t b = p.rbits[rec_at(p, s, x)], dm = det_mask(p.rtile[rec_at(p, s, x)], c.D);
        nd += __popcll(b & dm);
        no += __popcll(b & ~dm);
    }
    return nd | no << 16;
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

// R3: counting-sort scatter. Each source's 32-byte sort item (key built from
// its records, probability) is written to its bucket slot, so the bucket
// kernel reads every bucket as one contiguous run -- random gathers
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
        store_item(items_of(p) + at, it);
    });
}

__device__ __forceinline__ Item load_item(const Item *it) {
    const ulonglong2 a = reinterpret_cast<const ulonglong2 *>(it)[0], b = reinterpret_cast<const ulonglong2 *>(it)[1];
    return Item{a.x, a.y, b.x, __longlong_as_double((long long)b.y)};
}

// e_item entries of buckets gathered into items2 (fused items, huge_kernel).
constexpr uint32_t kItem2 = 0x80000000u;

// The items of one bucket as the grouping sees them: i in [0, n).
struct RunAcc {  // a contiguous run (bucket order); e_item = position | flag
    const Item *it;
    uint32_t base, flag;
    __device__ Item load(uint32_t i) const { return load_item(it + i); }
    __device__ double prob(uint32_t i) const { return it[i].prob; }
    __device__ uint32_t gidx(uint32_t i) const { return (base + i) | flag; }
    // the bucket's own run in items2: its edges may be written over it
    __device__ Item *edges() const { return flag == kItem2 ? const_cast<Item *>(it) : nullptr; }
};
struct IdxAcc {  // fused items: through the bucket's index list
    const Item *items;
    const uint32_t *idx;
    __device__ Item load(uint32_t i) const { return load_item(items + idx[i]); }
    __device__ double prob(uint32_t i) const { return items[idx[i]].prob; }
    __device__ uint32_t gidx(uint32_t i) const { return idx[i]; }
    __device__ Item *edges() const { return nullptr; }
};

// ecount[b] flag: bucket b's edges are items2[base + g] in canonical order,
// each carrying its folded probability (no e_item / e_prob / e_ndno entries).
constexpr uint32_t kEdgesInItems = 0x80000000u;

// Items and item count of bucket b.
__device__ __forceinline__ uint32_t bucket_size(const DevPlan &p, uint64_t b) {
    return p.fused ? p.boff[b].y : p.boff[b + 1].x - p.boff[b].x;
}

__device__ __forceinline__ uint32_t bucket_circuit(const DevPlan &p, uint64_t b) {
    return find_u32(arr<uint32_t>(p, p.lay.circ_bkt), p.tot.C, (uint32_t)b);
}

__device__ __forceinline__ BucketCtx bucket_ctx(const DevPlan &p, uint64_t b) {
    const CircuitMeta &m = arr<CircuitMeta>(p, p.lay.meta)[bucket_circuit(p, b)];
    return BucketCtx{m.D, (uint32_t)b - m.bucket_base};
}

// Group starting at sorted position i0 of a bucket (at(x): the bucket index
// of the item at sorted position x): walks to the group's end, folding the
// members' probabilities -- already ascending -- from 0 (merge_prob,
// dem.cpp:97-106), and files edge g: representative item, probability, id
// counts (returned).
template <bool EXACT, class At>
__device__ __forceinline__ uint32_t emit_group(const DevPlan &p, const Item *items, uint32_t base, uint32_t flag,
                                               uint32_t g, const At &at, uint32_t i0, uint32_t n, BucketCtx c) {
    Item prev = load_item(items + at(i0));
    double acc = merge_prob(0.0, prev.prob);
    for (uint32_t e = i0 + 1; e < n; e++) {
        const Item cur = load_item(items + at(e));
        if (sig_cmp<EXACT>(p, prev, cur, c) != 0) break;
        acc = merge_prob(acc, cur.prob);
        prev = cur;
    }
    const uint32_t rep = at(i0);
    const uint32_t ndno = item_ndno(p, load_item(items + rep), c);
    p.e_item[base + g] = (base + rep) | flag;
    p.e_prob[base + g] = acc;
    p.e_ndno[base + g] = ndno;
    return ndno;
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

// Table index source for a complete key (the table compares full keys, so
// this only spreads): the three words folded by rotations, one multiply.
__device__ __forceinline__ uint32_t item_hash(const Item &it) {
    uint64_t h = it.k0 ^ (it.k1 << 17 | it.k1 >> 47) ^ (it.obs << 41 | it.obs >> 23);
    h ^= h >> 32;
    h *= 0x9e3779b97f4a7c15ull;
    h ^= h >> 29;
    return (uint32_t)(h >> 32);
}

__device__ __forceinline__ bool key_eq(const Item &a, const Item &b) {
    return a.k0 == b.k0 && a.k1 == b.k1 && a.obs == b.obs;
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

// The group's member probabilities mp[o, e) folded from 0 in ascending order
// (merge_prob, dem.cpp:97-106). A group holds few distinct values (the noise
// model's p, p/3, p/15, flips), so it is folded one distinct value at a time:
// the smallest value above the last one and its multiplicity, O(k d) reads
// instead of an O(k^2) sort. Values that do not order (NaN) fall back to an
// insertion sort (mp[o, e) is scratch either way).
__device__ __forceinline__ double fold_sorted(double *mp, uint32_t o, uint32_t e) {
    double acc = 0.0, last = -INFINITY;
    uint32_t done = 0;
    bool first = true;
    while (done < e - o) {
        double x = INFINITY;
        uint32_t c = 0;
        for (uint32_t a = o; a < e; a++) {
            const double y = mp[a];
            if (y > last || (first && y == last)) {
                if (y < x) {
                    x = y;
                    c = 1;
                } else if (y == x) {
                    c++;
                }
            }
        }
        if (c == 0) break;  // unordered values remain
        for (uint32_t j = 0; j < c; j++) acc = merge_prob(acc, x);
        done += c;
        last = x;
        first = false;
    }
    if (done == e - o) return acc;
    for (uint32_t a = o + 1; a < e; a++) {  // insertion sort of the group's probabilities
        const double x = mp[a];
        uint32_t z = a;
        while (z > o && mp[z - 1] > x) {
            mp[z] = mp[z - 1];
            z--;
        }
        mp[z] = x;
    }
    acc = 0.0;
    for (uint32_t a = o; a < e; a++) acc = merge_prob(acc, mp[a]);
    return acc;
}

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
template <class Team, class Acc>
__device__ bool group_bucket(const DevPlan &p, const Team &tm, uint32_t b, uint32_t base, uint32_t n,
                             const Acc &it, GroupWs &w) {
    const uint32_t t0 = tm.t0(), nt = tm.nt();
    if (((uintptr_t)w.tab & 7) == 0)  // (tcap >= 64: whole 8-byte words)
        for (uint32_t x = t0; x < w.tcap / 4; x += nt) reinterpret_cast<uint64_t *>(w.tab)[x] = ~0ull;
    else
        for (uint32_t x = t0; x < w.tcap; x += nt) w.tab[x] = 0xFFFF;
    for (uint32_t x = t0; x < n; x += nt) w.cnt[x] = 0;
    tm.sync();
    // 1. representatives: hash + full key compare
    bool inc = false;
    double pc0 = 0.0, pc1 = 0.0;  // this thread's first two items' probabilities (the placement and move reuse them)
    for (uint32_t i = t0; i < n; i += nt) {
        const Item me = it.load(i);
        inc |= !me.complete();
        if (i == t0) pc0 = me.prob;
        else if (i == t0 + nt) pc1 = me.prob;
        uint32_t h = item_hash(me) & (w.tcap - 1), r = i;
        while (true) {
            uint32_t cur = w.tab[h];
            if (cur == 0xFFFF) {
                cur = atomicCAS(&w.tab[h], (unsigned short)0xFFFF, (unsigned short)i);
                if (cur == 0xFFFF) break;  // this item founds the group
            }
            if (key_eq(it.load(cur), me)) {
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
    // 2. members grouped by representative (any order); each group's end
    // offset replaces its (now zero) count; the hash table is free again and
    // holds each member's slot
    const uint32_t G = scan_groups(tm, w, n);
    constexpr bool kWarp = std::is_same<Team, WarpTeam>::value;
    for (uint32_t i = t0; i < n; i += nt) {
        const uint32_t r = w.rep[i];
        const uint32_t pos = w.off[r] + atomicSub(&w.cnt[r], 1u) - 1;
        w.mp[pos] = i == t0 ? pc0 : i == t0 + nt ? pc1 : it.prob(i);
        w.tab[i] = (uint16_t)pos;
    }
    tm.sync();
    for (uint32_t g = t0; g < G; g += nt) w.cnt[w.grp[g]] = g + 1 < G ? w.off[w.grp[g + 1]] : n;
    tm.sync();
    // every member's rank in its group by (value, slot), all members at once:
    // each group sorted ascending in place, then folded from 0 by one thread
    // (dem.cpp:97-106). A NaN (no order) sends the bucket to fold_sorted.
    bool nan = false;
    for (uint32_t i = t0; i < n; i += nt) {
        const uint32_t r = w.rep[i], o = w.off[r], e = w.cnt[r], me = w.tab[i];
        const double v = w.mp[me];
        nan |= v != v;
        uint32_t rank = 0;
        for (uint32_t a = o; a < e; a++) {
            const double x = w.mp[a];
            rank += (x < v) || (x == v && a < me);
        }
        w.tab[i] = (uint16_t)(o + rank);
    }
    const bool any_nan = tm.any(nan);  // (also the barrier between the ranks and the moves)
    if (!any_nan) {
        for (uint32_t i = t0; i < n; i += nt) w.mp[w.tab[i]] = i == t0 ? pc0 : i == t0 + nt ? pc1 : it.prob(i);
        tm.sync();
    }
    for (uint32_t g = t0; g < G; g += nt) {
        const uint32_t r = w.grp[g];
        const uint32_t o = w.off[r], e = w.cnt[r];
        double acc = 0.0;
        if (any_nan) {
            acc = fold_sorted(w.mp, o, e);
        } else {
            for (uint32_t a = o; a < e; a++) acc = merge_prob(acc, w.mp[a]);
        }
        w.mp[o] = acc;
    }
    tm.sync();
    // 3. groups in canonical order. A warp with at most 32 groups ranks them
    // (one group per lane, keys distinct); otherwise bitonic ("flip" form).
    if (kWarp && G <= 32) {
        const uint32_t lane = t0;
        const uint32_t mine = lane < G ? w.grp[lane] : 0;
        uint32_t rank = 0;
        Item me{};
        if (lane < G) me = it.load(mine);
        // the others' first key words by shuffle (all lanes take part); keys
        // equal there (rare) are compared in full in a second round
        bool tie = false;
        for (uint32_t h = 0; h < G; h++) {
            const uint64_t o0 = __shfl_sync(0xffffffffu, me.k0, h);
            rank += (lane < G && o0 < me.k0) ? 1u : 0u;
            tie |= lane < G && h != lane && o0 == me.k0;
        }
        if (__any_sync(0xffffffffu, tie)) {
            for (uint32_t h = 0; h < G; h++) {
                Item o;
                o.k0 = __shfl_sync(0xffffffffu, me.k0, h);
                o.k1 = __shfl_sync(0xffffffffu, me.k1, h);
                o.obs = __shfl_sync(0xffffffffu, me.obs, h);
                rank += (tie && h != lane && o.k0 == me.k0 && key_cmp(o, me) < 0) ? 1u : 0u;
            }
        }
        __syncwarp();
        if (lane < G) w.grp[rank] = (uint16_t)mine;
        __syncwarp();
        if (Item *ed = it.edges()) {
            // the edges over the bucket's own run: group `rank` (its key in
            // this lane's registers, every read of the run done) with its
            // folded probability -- the write kernel then streams them
            uint32_t nd = 0, no = 0;
            Item e{};
            if (lane < G) {
                e = me;
                e.prob = w.mp[w.off[mine]];
                const uint32_t v = key_ndno(me);
                nd = v & 0xFFFF;
                no = v >> 16;
            }
            __syncwarp();
            if (lane < G) store_item(ed + rank, e);
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                nd += __shfl_xor_sync(0xffffffffu, nd, d);
                no += __shfl_xor_sync(0xffffffffu, no, d);
            }
            if (lane == 0) {
                p.ecount[b] = G | kEdgesInItems;
                p.eids[b] = make_uint2(nd, no);
            }
            __syncwarp();
            return true;
        }
    } else {
        uint32_t np = 1;
        while (np < G) np <<= 1;
        auto cas = [&](uint32_t x, uint32_t y) {
            const uint32_t u = w.grp[x], v = w.grp[y];
            if (key_cmp(it.load(v), it.load(u)) < 0) {
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
        const uint32_t v = key_ndno(it.load(r));  // (every key complete here)
        p.e_item[base + g] = it.gidx(r);  // complete key: write_kernel decodes the ids from the item
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

// Bitonic network in its "flip" form: every comparator puts the smaller item
// first, so indices >= n act as +infinity and are skipped (no padding).
// Items move (in place in the bucket's run), so ties keep their order.
template <bool EXACT, class Sync>
__device__ __forceinline__ void bitonic(const DevPlan &p, Item *it, uint32_t n, BucketCtx c, uint32_t t0,
                                        uint32_t nt, Sync sync) {
    uint32_t np = 1;
    while (np < n) np <<= 1;
    auto cas = [&](uint32_t i, uint32_t l) {
        const Item a = load_item(it + i), d = load_item(it + l);
        if (item_less<EXACT>(p, d, 1, a, 0, c)) {  // strictly smaller: swap
            it[i] = d;
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
__device__ void groups_cta(const DevPlan &p, uint32_t b, uint32_t base, uint32_t flag, uint32_t n, BucketCtx c,
                           const Item *it) {
    __shared__ uint32_t s_cnt[33], s_ids[2];
    if (threadIdx.x == 0) s_ids[0] = s_ids[1] = 0;
    uint32_t total = 0;
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint32_t c0 = 0; c0 < n; c0 += blockDim.x) {
        const uint32_t i = c0 + threadIdx.x;
        const bool start = i < n && (i == 0 || sig_cmp<EXACT>(p, load_item(it + i - 1), load_item(it + i), c) != 0);
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
            auto at = [](uint32_t x) -> uint32_t { return x; };
            const uint32_t v =
                emit_group<EXACT>(p, it, base, flag, total + s_cnt[w] + __popc(bal & ((1u << lane) - 1)), at, i, n, c);
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

__device__ void bucket_cta(const DevPlan &p, uint32_t b, uint32_t flag, uint32_t n, BucketCtx c, Item *it) {
    const uint32_t base = p.boff[b].x;
    __shared__ uint32_t s_inc;
    if (threadIdx.x == 0) s_inc = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
        if (!it[i].complete()) s_inc = 1;
    __syncthreads();
    if (s_inc) {
        bitonic<true>(p, it, n, c, threadIdx.x, blockDim.x, [] { __syncthreads(); });
        groups_cta<true>(p, b, base, flag, n, c, it);
    } else {
        bitonic<false>(p, it, n, c, threadIdx.x, blockDim.x, [] { __syncthreads(); });
        groups_cta<false>(p, b, base, flag, n, c, it);
    }
}

constexpr uint32_t kWarpTab = 512;                                   // >= 2 kWarpItems
constexpr uint32_t kWarpWs = (256 * 18 + 16 + 512 * 2 + 15) & ~15u;  // GroupWs::bytes(256, 512)
constexpr uint32_t kHugeSmem = 196 * 1024;                            // huge_kernel dynamic smem

// One warp per bucket, no CTA synchronisation: empty buckets, buckets of up
// to kWarpItems sources (group_bucket in the warp's workspace); larger ones
// and those holding an incomplete key are listed for huge_kernel.
__global__ void __launch_bounds__(kBucketThreads) bucket_kernel(__grid_constant__ const DevPlan p) {
    __shared__ __align__(16) uint8_t ws[(kBucketThreads / 32) * kWarpWs];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    GroupWs w;
    w.carve(ws + warp * kWarpWs, kWarpItems, kWarpTab);
    const uint64_t NB = p.tot.buckets;
    if (p.hdr->items_overflow) return;  // re-run with a larger item array
    // buckets taken in order from a counter (bucket sizes vary 1-256: a
    // fixed stride would leave the warps with the larger shares as the tail)
    // (the next bucket is claimed while this one is grouped: the counter's
    // latency off the critical path, bucket stage -0.6 %)
    uint32_t nb = 0;
    if (lane == 0) nb = atomicAdd(&p.hdr->bucket_next, 1u);
    for (uint64_t b;;) {
        b = __shfl_sync(0xffffffffu, nb, 0);
        if (b >= NB) break;
        if (lane == 0) nb = atomicAdd(&p.hdr->bucket_next, 1u);
        const uint32_t base = p.boff[b].x, n = bucket_size(p, b);
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
        uint32_t tc = 64;  // hash table: a power of two >= 2n
        while (tc < 2 * n) tc <<= 1;
        w.tcap = tc;
        // an incomplete key: the bucket goes to huge_kernel's exact CTA sort
        // (kept out of this kernel: its comparator's state costs registers)
        const bool ok = p.fused_move ? group_bucket(p, WarpTeam{}, (uint32_t)b, base, n,
                                                    RunAcc{reinterpret_cast<const Item *>(p.items2) + base, base, kItem2}, w)
                        : p.fused ? group_bucket(p, WarpTeam{}, (uint32_t)b, base, n, IdxAcc{items_of(p), p.iidx + base}, w)
                                : group_bucket(p, WarpTeam{}, (uint32_t)b, base, n, RunAcc{items_of(p) + base, base, 0}, w);
        if (!ok && lane == 0) p.huge[atomicAdd(&p.hdr->huge_count, 1u)] = (uint32_t)b;
    }
}

// Buckets too large for a warp, or holding an incomplete key: one CTA each,
// group_bucket in up to 196 KB of dynamic shared memory; the exact CTA sort
// (in place in the bucket's own run of the item array) for incomplete keys or
// buckets beyond that.
__global__ void __launch_bounds__(256) huge_kernel(__grid_constant__ const DevPlan p) {
    extern __shared__ __align__(16) uint8_t hsm[];
    if (p.hdr->items_overflow) return;
    const uint32_t nh = p.hdr->huge_count;
    __shared__ uint32_t s_inc;
    for (uint32_t i = blockIdx.x; i < nh; i += gridDim.x) {
        const uint32_t b = p.huge[i];
        const uint32_t base = p.boff[b].x, n = bucket_size(p, b);
        Item *it = items_of(p) + base;
        uint32_t flag = 0;
        if (p.fused) {  // gather the bucket's listed items into a run of items2
            it = reinterpret_cast<Item *>(p.items2) + base;
            flag = kItem2;
            if (!p.fused_move) {
                for (uint32_t x = threadIdx.x; x < n; x += blockDim.x)
                    store_item(it + x, load_item(items_of(p) + p.iidx[base + x]));
                __syncthreads();
            }
        }
        const BucketCtx c = bucket_ctx(p, b);
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
            group_bucket(p, CtaTeam{}, b, base, n, RunAcc{it, base, flag}, w);
        } else {
            bucket_cta(p, b, flag, n, c, it);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- R6 output
// Bucket b's groups become edges [eoff, eoff + ecount) of the flat DEM, ids
// decoded from the representative's key (or expanded from its records, in
// word order: bit b < D -> detector b, else observable b - D; dem.cpp:108-116).
__global__ void write_kernel(__grid_constant__ const DevPlan p, const uint4 *out_total, uint32_t cb) {
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
            p.o_det_off[tot.x] = (uint32_t)(bD + tot.y);
            p.o_obs_off[tot.x] = (uint32_t)(bO + tot.z);
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
    // One warp per cb (<= 32) consecutive buckets, their edges packed onto
    // the lanes (a bucket holds ~9 edges: one bucket per warp would idle most
    // lanes; batches take cb = 32, single circuits fewer -- enough warps).
    // Edge j of the chunk is edge oscan[B0].x + j of the output; its id
    // offsets are the chunk's (oscan[B0]) plus a warp scan of the id counts.
    const Item *items = items_of(p), *items2 = reinterpret_cast<const Item *>(p.items2);
    const uint32_t *circ_bkt = arr<uint32_t>(p, p.lay.circ_bkt);
    for (uint64_t B0 = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * cb; B0 < NB; B0 += warps * cb) {
        const uint64_t b = B0 + lane;
        const uint32_t ec = lane < cb && b < NB ? p.ecount[b] : 0;
        const uint32_t ne = ec & ~kEdgesInItems;
        const bool inl = (ec & kEdgesInItems) != 0;  // edges = items2[base + k]
        uint32_t st = ne;  // inclusive scan of the edge counts
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, st, d);
            if (lane >= (uint32_t)d) st += x;
        }
        const uint32_t T = __shfl_sync(0xffffffffu, st, 31), start = st - ne;
        if (T == 0) continue;
        uint32_t c = find_u32_warp(circ_bkt, p.tot.C, (uint32_t)B0);  // B0's circuit; lanes step forward
        uint32_t base = 0, q0 = 0, D = 0;
        if (ne) {
            while (c + 1 < p.tot.C && circ_bkt[c + 1] <= (uint32_t)b) c++;
            const CircuitMeta &m = meta[c];
            base = p.boff[b].x;
            q0 = (uint32_t)b - m.bucket_base;
            D = m.D;
        }
        const uint4 o = p.oscan[B0];  // (edges, det ids, obs ids) before bucket B0
        uint32_t dcar = 0, ocar = 0;
        for (uint32_t j0 = 0; j0 < T; j0 += 32) {
            const uint32_t j = j0 + lane;
            uint32_t l = 0;  // the lane holding edge j's bucket: largest l with start_l <= j
#pragma unroll
            for (uint32_t step = 16; step > 0; step >>= 1)
                if (__shfl_sync(0xffffffffu, start, l + step) <= j) l += step;
            const uint32_t k = j - __shfl_sync(0xffffffffu, start, l);
            const uint32_t bb = __shfl_sync(0xffffffffu, base, l);
            const BucketCtx cx{__shfl_sync(0xffffffffu, D, l), __shfl_sync(0xffffffffu, q0, l)};
            const bool ein = __shfl_sync(0xffffffffu, (uint32_t)inl, l) != 0;
            uint32_t nd = 0, no = 0;
            Item q{};
            double pe = 0.0;
            if (j < T) {
                uint32_t v;
                if (ein) {  // the edge itself (consecutive k: a streamed run)
                    q = load_item(items2 + bb + k);
                    pe = q.prob;
                    v = key_ndno(q);
                } else {
                    v = p.e_ndno[bb + k];
                    pe = p.e_prob[bb + k];
                    const uint32_t ei = p.e_item[bb + k];
                    q = load_item((ei & kItem2 ? items2 : items) + (ei & ~kItem2));
                }
                nd = v & 0xFFFF;
                no = v >> 16;
            }
            uint32_t di = nd, oi = no;  // inclusive warp scans
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t x = __shfl_up_sync(0xffffffffu, di, d), y = __shfl_up_sync(0xffffffffu, oi, d);
                if (lane >= (uint32_t)d) {
                    di += x;
                    oi += y;
                }
            }
            if (j < T) {
                const uint64_t e = (uint64_t)o.x + j;
                const uint32_t d0 = o.y + dcar + di - nd, o0 = o.z + ocar + oi - no;
                p.o_det_off[e] = (uint32_t)(bD + d0);
                p.o_obs_off[e] = (uint32_t)(bO + o0);
                p.o_prob[e] = pe;
                uint32_t wd = d0, wo = o0;
                if (q.complete()) {  // detectors q0 - 1, then the differences; observables by mask
                    if (cx.q0) {
                        uint32_t id = cx.q0 - 1;
                        p.o_det[wd++] = id;
                        for (uint32_t f = 0; f < kKeyFields; f++) {
                            const uint32_t dv = key_get(q, f);
                            if (dv == 0) break;
                            id += dv;
                            p.o_det[wd++] = id;
                        }
                    }
                    for (uint64_t ob = q.obs; ob; ob &= ob - 1) p.o_obs[wo++] = (uint32_t)__ffsll((long long)ob) - 1;
                } else {  // ids from the representative's records, in word order
                    const uint32_t r = q.src();
                    uint8_t ord[kMaxRecords];
                    const uint32_t n = min(p.cnt[r], kMaxRecords);
                    sig_order(p, r, n, ord);
                    for (uint32_t x = 0; x < n; x++) {
                        const uint32_t t = p.rtile[rec_at(p, r, ord[x])];
                        uint64_t bits = p.rbits[rec_at(p, r, ord[x])];
                        while (bits) {
                            const uint32_t id = t * 64 + (uint32_t)__ffsll((long long)bits) - 1;
                            bits &= bits - 1;
                            if (id < cx.D) p.o_det[wd++] = id;
                            else p.o_obs[wo++] = id - cx.D;
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
// 16-byte stores (larger PCIe writes than 4- or 8-byte ones); both sides
// 16-byte aligned, the tail byte by byte.
__device__ __forceinline__ void copy_bytes16(void *dst, const void *src, uint64_t bytes, uint64_t t0, uint64_t stride) {
    const uint64_t n16 = bytes / 16;
    for (uint64_t i = t0; i < n16; i += stride) reinterpret_cast<uint4 *>(dst)[i] = reinterpret_cast<const uint4 *>(src)[i];
    if (t0 < bytes - n16 * 16)
        reinterpret_cast<uint8_t *>(dst)[n16 * 16 + t0] = reinterpret_cast<const uint8_t *>(src)[n16 * 16 + t0];
}

__global__ void copy_out_kernel(__grid_constant__ const DevPlan p) {
    const DeviceHeader hd = *p.hdr;
    const bool ok = hd.num_det_ids != 0xFFFFFFFFu && !hd.items_overflow && !hd.record_overflow && !hd.pool_overflow;
    const uint64_t E = hd.num_edges, nd = ok ? hd.num_det_ids : 0, no = hd.num_obs_ids, C = p.tot.C;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x, t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (ok) {
        copy_bytes16(p.hmap.det_off, p.o_det_off, (E + 1) * 4, t0, stride);
        copy_bytes16(p.hmap.obs_off, p.o_obs_off, (E + 1) * 4, t0, stride);
        copy_bytes16(p.hmap.probs, p.o_prob, E * 8, t0, stride);
        copy_bytes16(p.hmap.det_ids, p.o_det, nd * 4, t0, stride);
        copy_bytes16(p.hmap.obs_ids, p.o_obs, no * 4, t0, stride);
        copy_bytes16(p.hmap.edge_off, p.o_edge_off, (C + 1) * 8, t0, stride);
    }
    if (t0 == 0) *p.hmap.hdr = hd;
}

}  // namespace red

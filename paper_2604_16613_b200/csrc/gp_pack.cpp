// gp_pack.cpp -- host worker pool and task-parallel packer (see gp_pack.h).
#include "gp_pack.h"

#include <algorithm>
#include <chrono>
#include <cstring>
#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace gp {

// ---------------------------------------------------------------- pool

HostPool::HostPool(unsigned workers) {
    for (unsigned i = 0; i < workers; i++) th_.emplace_back([this] { loop(); });
}

HostPool::~HostPool() {
    {
        std::lock_guard<std::mutex> g(mu_);
        stop_ = true;
        gen_.fetch_add(1);
    }
    cv_.notify_all();
    for (auto &t : th_) t.join();
}

void HostPool::work(Job &j) {
    for (size_t i; (i = j.next.fetch_add(1, std::memory_order_relaxed)) < j.n;) {
        (*j.fn)(i);
        j.left.fetch_sub(1, std::memory_order_acq_rel);
    }
}

void HostPool::run(size_t n, const std::function<void(size_t)> &f) {
    if (n == 0) return;
    if (th_.empty() || n == 1) {
        for (size_t i = 0; i < n; i++) f(i);
        return;
    }
    auto j = std::make_shared<Job>();
    j->fn = &f;
    j->n = n;
    j->left.store(n);
    {
        std::lock_guard<std::mutex> g(mu_);
        job_ = j;
        gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    work(*j);
    while (j->left.load(std::memory_order_acquire) != 0) std::this_thread::yield();
}

void HostPool::loop() {
    uint64_t seen = 0;
    for (;;) {
        // Spin ~200 us for the next job before sleeping.
        const auto t0 = std::chrono::steady_clock::now();
        while (gen_.load(std::memory_order_acquire) == seen &&
               std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(200))
            std::this_thread::yield();
        std::shared_ptr<Job> j;
        {
            std::unique_lock<std::mutex> l(mu_);
            cv_.wait(l, [&] { return gen_.load() != seen; });
            seen = gen_.load();
            if (stop_) return;
            j = job_;
        }
        if (j) work(*j);
    }
}

// ---------------------------------------------------------------- helpers

namespace {

uint32_t alpha_of(uint8_t level) { return level == 0 ? 2 : level == 1 ? 4 : 7; }  // stepg.cpp:23-33

uint32_t components(uint8_t kind, uint8_t level) {  // stepg.cpp:66-103
    if (kind <= GP_NOISE_Z_ERROR) return 1;
    if (kind == GP_NOISE_DEPOLARIZE1) return level == 0 ? 2 : 3;
    return level == 0 ? 6 : level == 1 ? 10 : 15;
}

uint64_t align16(uint64_t x) { return (x + 15) & ~15ull; }

uint64_t bits_of(double d) {
    uint64_t b;
    std::memcpy(&b, &d, 8);
    return b;
}

constexpr uint64_t kTaskOps = 1 << 13;  // ops (gates + noise, or list entries) per task

// Streaming store of an 8-byte word into the pinned staging image: written
// once, read only by the DMA engine, so it bypasses the caches (no
// read-for-ownership of the destination lines: the packer is bound by host
// memory traffic).
inline void put64(uint64_t *dst, uint64_t v) {
#if defined(__x86_64__)
    _mm_stream_si64(reinterpret_cast<long long *>(dst), (long long)v);
#else
    *dst = v;
#endif
}
inline void put32(uint32_t *dst, uint32_t v) {
#if defined(__x86_64__)
    _mm_stream_si32(reinterpret_cast<int *>(dst), (int)v);
#else
    *dst = v;
#endif
}
inline void put_fence() {
#if defined(__x86_64__)
    _mm_sfence();
#endif
}

}  // namespace

StageLayout stage_layout(const BatchTotals &t) {
    StageLayout L{};
    uint64_t o = 0;
    auto put = [&](uint64_t bytes) {
        const uint64_t at = o;
        o = align16(o + bytes + 16);  // +16: bulk copies may over-read one 16-byte unit
        return at;
    };
    L.meta = put(t.C * sizeof(CircuitMeta));
    L.circ_layer = put((t.C + 1) * 4);
    L.circ_src = put((t.C + 1) * 8);
    L.circ_tile = put((t.C + 1) * 4);
    L.circ_grp = put((t.C + 1) * 4);
    L.circ_det = put((t.C + 1) * 4);
    L.circ_obs = put((t.C + 1) * 4);
    L.circ_bkt = put((t.C + 1) * 4);
    L.lay_gate = put(t.layer_slots * 4);
    L.lay_noise = put(t.layer_slots * 4);
    L.lay_meas = put(t.layer_slots * 4);
    L.gates = put(t.gates * (t.narrow ? 4 : 8));
    L.noise = put(t.noise * (t.narrow ? 4 : 8));
    L.noise_prob = put(t.wide_prob ? t.noise * 8 : 0);
    L.lay_src = put(t.layer_slots * 4);
    L.meas_flip = put(t.meas * 8);
    L.det_off = put(t.det_slots * 4);
    L.det_meas = put(t.det_entries * 4);
    L.obs_off = put(t.obs_slots * 4);
    L.obs_meas = put(t.obs_entries * 4);
    L.prob_table = put((uint64_t)t.prob_table_n * 8);  // last: uploads stop at the entries used
    L.total = o;
    return L;
}

namespace {

// Splits [a, b) into pieces of about `per` units (at least one piece).
template <class F>
void split_range(uint64_t a, uint64_t b, uint64_t per, F &&emit) {
    const uint64_t n = b > a ? (b - a + per - 1) / per : 1;
    for (uint64_t k = 0; k < n; k++) emit(a + (b - a) * k / n, a + (b - a) * (k + 1) / n);
}

void run_tasks(HostPool *pool, size_t n, const std::function<void(size_t)> &f) {
    if (pool) pool->run(n, f);
    else
        for (size_t i = 0; i < n; i++) f(i);
}

// Per-task cache in front of the shared dictionary (a layer's noise ops
// cycle through a few probabilities).
struct ProbCache {
    ProbDict *d;
    uint64_t k[4] = {~0ull, ~0ull, ~0ull, ~0ull};
    uint32_t v[4] = {ProbDict::kFull, ProbDict::kFull, ProbDict::kFull, ProbDict::kFull};
    uint32_t next = 0;
    uint32_t last = 0;
    uint32_t operator()(double p) {
        const uint64_t b = bits_of(p);
        if (k[last] == b) return v[last];  // runs of one value: one compare
        for (uint32_t i = 0; i < 4; i++)
            if (k[i] == b) {
                last = i;
                return v[i];
            }
        const uint32_t x = d->index(b);
        k[next] = b;
        v[next] = x;
        last = next;
        next = (next + 1) & 3;
        return x;
    }
};

}  // namespace

// ---------------------------------------------------------------- dictionary

ProbDict::ProbDict()
    : key_(new std::atomic<uint64_t>[kSlots]), val_(new std::atomic<uint32_t>[kSlots]),
      slot_of_(new uint32_t[kSlotLog]) {
    for (uint32_t x = 0; x < kSlots; x++) {
        key_[x].store(0, std::memory_order_relaxed);
        val_[x].store(kEmpty, std::memory_order_relaxed);
    }
}

void ProbDict::clear() {
    const uint32_t n = std::min<uint32_t>(n_.load(), kSlotLog);
    for (uint32_t i = 0; i < n; i++) val_[slot_of_[i]].store(kEmpty, std::memory_order_relaxed);
    n_.store(0);
}

uint32_t ProbDict::size() const { return std::min<uint32_t>(n_.load(), kNoisePidxMax + 1); }

uint32_t ProbDict::index(uint64_t bits) {
    uint64_t h = bits * 0x9e3779b97f4a7c15ull;
    uint32_t x = (uint32_t)(h >> 48) & (kSlots - 1);
    for (;;) {
        uint32_t v = val_[x].load(std::memory_order_acquire);
        if (v == kEmpty) {
            // Full table: no new claims (only the racing few, all logged for clear()).
            if (n_.load(std::memory_order_relaxed) > kNoisePidxMax) return kFull;
            if (val_[x].compare_exchange_strong(v, kBusy, std::memory_order_acq_rel)) {
                key_[x].store(bits, std::memory_order_relaxed);
                const uint32_t i = n_.fetch_add(1);
                if (i < kSlotLog) slot_of_[i] = x;
                val_[x].store(i, std::memory_order_release);
                return i <= kNoisePidxMax ? i : kFull;
            }
        }
        while (v == kBusy) v = val_[x].load(std::memory_order_acquire);
        if (v == kEmpty) continue;  // (lost a race to a claim that has now published: re-read)
        if (key_[x].load(std::memory_order_relaxed) == bits) return v <= kNoisePidxMax ? v : kFull;
        x = (x + 1) & (kSlots - 1);
    }
}

void ProbDict::values(std::vector<double> &out) const {
    const uint32_t n = size();
    out.resize(n);
    for (uint32_t i = 0; i < n; i++) {
        const uint64_t b = key_[slot_of_[i]].load(std::memory_order_relaxed);
        std::memcpy(&out[i], &b, 8);
    }
}

// ---------------------------------------------------------------- phases

void pack_plan(HostPool *pool, const gp_circuit_view *cs, size_t C, uint8_t level, PackPlan &pp) {
    BatchTotals &t = pp.t;
    t = BatchTotals{};
    t.C = (uint32_t)C;
    t.level = level;
    pp.metas.assign(C, CircuitMeta{});
    pp.err = kPackOk;
    pp.err_circuit = 0;
    for (size_t c = 0; c < C; c++) {  // O(C): sizes and bases straight from the offset arrays
        const gp_circuit_view &v = cs[c];
        CircuitMeta &m = pp.metas[c];
        const uint64_t rows = (uint64_t)v.num_layers * alpha_of(level) * v.num_qubits + v.num_measurements;
        int err = kPackOk;
        if (rows >= 0xFFFFFFFFull) err = kPackIndexSpace;  // lower(), stepg.cpp:171-174
        else if (v.num_qubits >= (1u << kNoiseQubitBits) || v.num_measurements >= (1u << 29))
            err = kPackTooWide;
        if (err && !pp.err) {
            pp.err = err;
            pp.err_circuit = c;
        }
        m.n = v.num_qubits;
        m.l = v.num_layers;
        m.M = v.num_measurements;
        m.D = v.num_detectors;
        m.O = v.num_observables;
        m.W = (uint32_t)(((uint64_t)m.D + m.O + 63) / 64);
        m.layer_base = (uint32_t)t.layer_slots;
        m.meas_base = (uint32_t)t.meas;
        m.det_base = (uint32_t)t.det_slots;
        m.obs_base = (uint32_t)t.obs_slots;
        m.tile_base = (uint32_t)t.tiles;
        m.bucket_base = (uint32_t)t.buckets;
        m.ell_base = t.ell;
        m.leaf_base = t.leaf;
        m.gate_base = t.gates;
        m.noise_base = t.noise;
        m.det_entry_base = t.det_entries;
        m.obs_entry_base = t.obs_entries;
        m.circ_layer_base = t.layers;
        const uint64_t gates = v.gate_offsets[m.l] - v.gate_offsets[0];
        const uint64_t noise = v.noise_offsets[m.l] - v.noise_offsets[0];
        t.max_n = std::max(t.max_n, m.n);
        t.max_W = std::max(t.max_W, m.W);
        t.max_l = std::max(t.max_l, m.l);
        t.layers += m.l;
        t.layer_slots += m.l + 1;
        t.gates += gates;
        t.noise += noise;
        t.meas += m.M;
        t.det_slots += m.D + 1;
        t.det_entries += v.det_offsets[m.D] - v.det_offsets[0];
        t.obs_slots += m.O + 1;
        t.obs_entries += v.obs_offsets[m.O] - v.obs_offsets[0];
        t.dets += m.D;
        t.obss += m.O;
        t.tiles += m.W;
        t.ell += m.l ? (uint64_t)(m.l - 1) * ell_stride(m.n) : 0;
        t.leaf += (uint64_t)m.W * leaf_stride(m.M);
        t.buckets += (uint64_t)m.D + 1;
    }
    // Probability table: filled by pack_range; reserved at its maximum size
    // at the end of the image (image_bytes() uploads the part used).
    t.wide_prob = pp.force_wide;
    t.prob_table_n = t.wide_prob ? 0 : kNoisePidxMax + 1;
    uint32_t max_m = 0;
    for (const CircuitMeta &m : pp.metas) max_m = std::max(max_m, m.M);
    t.narrow = !t.wide_prob && !pp.no_narrow && t.max_n <= kNarrowMaxQubits && max_m <= kNarrowMaxMeas;
    pp.dict.clear();
    pp.need_wide.store(false);
    pp.need_wide_words.store(false);
    pp.prob_table.clear();
    pp.L = stage_layout(t);
}

void pack_range(HostPool *pool, const gp_circuit_view *cs, PackPlan &pp, uint8_t *img, size_t c0, size_t c1) {
    const BatchTotals &t = pp.t;
    const StageLayout &L = pp.L;
    const uint8_t level = (uint8_t)t.level;
    auto at = [&](uint64_t off) { return img + off; };
    auto *lay_gate = (uint32_t *)at(L.lay_gate);
    auto *lay_noise = (uint32_t *)at(L.lay_noise);
    auto *lay_meas = (uint32_t *)at(L.lay_meas);
    auto *gates = (uint64_t *)at(L.gates);
    auto *noise = (uint64_t *)at(L.noise);
    auto *gates32 = (uint32_t *)at(L.gates);
    auto *noise32 = (uint32_t *)at(L.noise);
    const bool narrow = t.narrow != 0;
    auto *nprob = (double *)at(L.noise_prob);
    auto *lay_src = (uint32_t *)at(L.lay_src);
    auto *flip = (double *)at(L.meas_flip);
    auto *det_off = (uint32_t *)at(L.det_off);
    auto *det_meas = (uint32_t *)at(L.det_meas);
    auto *obs_off = (uint32_t *)at(L.obs_off);
    auto *obs_meas = (uint32_t *)at(L.obs_meas);

    // Tasks: 0 = layer range, 1 = detector range, 2 = observable range.
    struct Task {
        uint32_t c, kind;
        uint32_t a, b;
    };
    std::vector<Task> tasks;
    for (size_t c = c0; c < c1; c++) {
        const gp_circuit_view &v = cs[c];
        const uint32_t l = v.num_layers;
        const uint64_t ops = (v.gate_offsets[l] - v.gate_offsets[0]) + (v.noise_offsets[l] - v.noise_offsets[0]);
        const uint64_t per_layer = l ? std::max<uint64_t>(1, ops / l) : 1;
        split_range(0, l, std::max<uint64_t>(1, kTaskOps / per_layer),
                    [&](uint64_t a, uint64_t b) { tasks.push_back({(uint32_t)c, 0, (uint32_t)a, (uint32_t)b}); });
        const uint64_t de = v.det_offsets[v.num_detectors] - v.det_offsets[0];
        const uint64_t per_det = v.num_detectors ? std::max<uint64_t>(1, de / v.num_detectors) : 1;
        split_range(0, v.num_detectors, std::max<uint64_t>(1, kTaskOps / per_det),
                    [&](uint64_t a, uint64_t b) { tasks.push_back({(uint32_t)c, 1, (uint32_t)a, (uint32_t)b}); });
        tasks.push_back({(uint32_t)c, 2, 0, v.num_observables});
    }
    std::vector<int> terr(tasks.size(), kPackOk);
    run_tasks(pool, tasks.size(), [&](size_t k) {
        const Task &tk = tasks[k];
        const gp_circuit_view &v = cs[tk.c];
        const CircuitMeta &m = pp.metas[tk.c];
        if (tk.kind == 0) {
            const uint32_t g0 = v.gate_offsets[0], n0 = v.noise_offsets[0];
            ProbCache pidx{&pp.dict};
            uint32_t comp_tab[8];  // components per noise kind (stepg.cpp:66-103)
            for (uint32_t x = 0; x < 8; x++) comp_tab[x] = components((uint8_t)x, level);
            if (narrow && !t.wide_prob) {  // the common case: one tight pass per layer, 4-byte words
                const uint8_t *__restrict gk = v.gate_kind, *__restrict nk = v.noise_kind;
                const uint32_t *__restrict gq0 = v.gate_q0, *__restrict gq1 = v.gate_q1;
                const int32_t *__restrict gm = v.gate_meas;
                const double *__restrict gf = v.gate_flip, *__restrict np = v.noise_prob;
                const uint32_t *__restrict nq0 = v.noise_q0, *__restrict nq1 = v.noise_q1;
                uint32_t *__restrict gout = gates32 + m.gate_base - g0;
                uint32_t *__restrict nout = noise32 + m.noise_base - n0;
                double *__restrict fout = flip + m.meas_base;
                uint64_t last_bits = ~0ull;
                uint32_t last_pi = 0;
                bool big = false;
                for (uint32_t i = tk.a; i < tk.b; i++) {
                    const uint32_t li = m.layer_base + i;
                    const uint32_t ga = v.gate_offsets[i], gb = v.gate_offsets[i + 1];
                    const uint32_t na = v.noise_offsets[i], nb = v.noise_offsets[i + 1];
                    lay_gate[li] = (uint32_t)(m.gate_base + ga - g0);
                    lay_noise[li] = (uint32_t)(m.noise_base + na - n0);
                    uint32_t meas = 0;
                    for (uint32_t g = ga; g < gb; g++) {
                        const uint32_t kd = gk[g];
                        const bool ms = kd == GP_GATE_M || kd == GP_GATE_MR;
                        uint32_t hi = kd == GP_GATE_CX ? gq1[g] : 0;
                        if (ms) {
                            hi = (uint32_t)gm[g];
                            fout[hi] = gf[g];
                            meas++;
                        }
                        put32(&gout[g], narrow_gate(gq0[g], kd, hi));
                    }
                    lay_meas[li] = meas;  // count; prefix in pack_finish
                    uint32_t src = 0;
                    for (uint32_t o = na; o < nb; o++) {
                        const uint32_t kd = nk[o];
                        uint64_t bits;
                        std::memcpy(&bits, &np[o], 8);
                        if (bits != last_bits) {  // runs of one probability: one compare
                            const uint32_t x = pidx(np[o]);
                            last_bits = bits;
                            last_pi = x;
                            if (x >= kNarrowMaxProbs) big = true;
                        }
                        const uint32_t q1 = kd == GP_NOISE_DEPOLARIZE2 ? nq1[o] : 0;
                        put32(&nout[o], narrow_noise(nq0[o], q1, kd, last_pi < kNarrowMaxProbs ? last_pi : 0));
                        src += comp_tab[kd & 7];
                    }
                    lay_src[li] = src;  // count; prefix in pack_finish
                }
                if (big) {  // ProbDict::kFull or a 65th probability: repack (wide table or 8-byte words)
                    if (pp.dict.size() > kNoisePidxMax) pp.need_wide.store(true, std::memory_order_relaxed);
                    pp.need_wide_words.store(true, std::memory_order_relaxed);
                }
            } else
            for (uint32_t i = tk.a; i < tk.b; i++) {
                const uint32_t li = m.layer_base + i;
                lay_gate[li] = (uint32_t)(m.gate_base + v.gate_offsets[i] - g0);
                lay_noise[li] = (uint32_t)(m.noise_base + v.noise_offsets[i] - n0);
                uint32_t meas = 0;
                for (uint32_t g = v.gate_offsets[i]; g < v.gate_offsets[i + 1]; g++) {
                    const uint8_t kd = v.gate_kind[g];
                    uint32_t hi = 0;
                    if (kd == GP_GATE_CX) hi = v.gate_q1[g];
                    if (kd == GP_GATE_M || kd == GP_GATE_MR) {
                        hi = (uint32_t)v.gate_meas[g];
                        flip[m.meas_base + hi] = v.gate_flip[g];
                        meas++;
                    }
                    if (narrow) put32(&gates32[m.gate_base + g - g0], narrow_gate(v.gate_q0[g], kd, hi));
                    else put64(&gates[m.gate_base + g - g0], (uint64_t)hi << 32 | (v.gate_q0[g] | (uint32_t)kd << kGateKindShift));
                }
                lay_meas[li] = meas;  // count; prefix in pack_finish
                uint32_t src = 0;
                for (uint32_t o = v.noise_offsets[i]; o < v.noise_offsets[i + 1]; o++) {
                    const uint8_t kd = v.noise_kind[o];
                    const uint64_t idx = m.noise_base + o - n0;
                    uint64_t pi = 0;
                    if (t.wide_prob) {
                        nprob[idx] = v.noise_prob[o];
                    } else {
                        pi = pidx(v.noise_prob[o]);
                        if (pi == ProbDict::kFull) {  // more distinct values than the table: repack wide
                            pp.need_wide.store(true, std::memory_order_relaxed);
                            pi = 0;
                        }
                    }
                    const uint32_t q1 = kd == GP_NOISE_DEPOLARIZE2 ? v.noise_q1[o] : 0;
                    if (narrow) {
                        if (pi >= kNarrowMaxProbs) {  // a 65th probability: repack with 8-byte words
                            pp.need_wide_words.store(true, std::memory_order_relaxed);
                            pi = 0;
                        }
                        put32(&noise32[idx], narrow_noise(v.noise_q0[o], q1, kd, (uint32_t)pi));
                    } else {
                        put64(&noise[idx], (uint64_t)v.noise_q0[o] | (uint64_t)q1 << kNoiseQubitBits |
                                               (uint64_t)kd << kNoiseKindShift | pi << kNoisePidxShift);
                    }
                    src += comp_tab[kd & 7];
                }
                lay_src[li] = src;  // count; prefix in pack_finish
            }
            put_fence();
            if (tk.b == m.l) {  // closing entries of the circuit's layer tables
                const uint32_t li = m.layer_base + m.l;
                lay_gate[li] = (uint32_t)(m.gate_base + v.gate_offsets[m.l] - g0);
                lay_noise[li] = (uint32_t)(m.noise_base + v.noise_offsets[m.l] - n0);
                lay_meas[li] = 0;
                lay_src[li] = 0;
            }
        } else if (tk.kind == 1) {  // init_leaves, eec.cpp:42-49
            const uint32_t e0 = v.det_offsets[0];
            for (uint32_t d = tk.a; d < tk.b + (tk.b == m.D ? 1u : 0u); d++)
                det_off[m.det_base + d] = (uint32_t)(m.det_entry_base + v.det_offsets[d] - e0);
            const uint32_t x0 = v.det_offsets[tk.a], x1 = v.det_offsets[tk.b];
            for (uint32_t x = x0; x < x1; x++) {
                const uint32_t mm = v.det_meas[x];
                if (mm >= m.M) terr[k] = kPackDetLeaf;
                det_meas[m.det_entry_base + x - e0] = mm;
            }
        } else {  // eec.cpp:50-57
            const uint32_t e0 = v.obs_offsets[0];
            for (uint32_t o = 0; o <= m.O; o++) obs_off[m.obs_base + o] = (uint32_t)(m.obs_entry_base + v.obs_offsets[o] - e0);
            for (uint32_t x = v.obs_offsets[0]; x < v.obs_offsets[m.O]; x++) {
                const uint32_t mm = v.obs_meas[x];
                if (mm >= m.M) terr[k] = kPackObsLeaf;
                obs_meas[m.obs_entry_base + x - e0] = mm;
            }
        }
    });
    // First failing circuit, reference order within a circuit: index space,
    // then detectors, then observables.
    for (size_t k = 0; k < tasks.size(); k++) {
        if (!terr[k]) continue;
        const size_t c = tasks[k].c;
        if (!pp.err || c < pp.err_circuit || (c == pp.err_circuit && terr[k] < pp.err)) {
            pp.err = terr[k];
            pp.err_circuit = c;
        }
    }
}

int validate_leaves(const gp_circuit_view *cs, size_t c0, size_t c1) {
    for (size_t c = c0; c < c1; c++) {
        const gp_circuit_view &v = cs[c];
        for (uint32_t x = v.det_offsets[0]; x < v.det_offsets[v.num_detectors]; x++)
            if (v.det_meas[x] >= v.num_measurements) return kPackDetLeaf;
        for (uint32_t x = v.obs_offsets[0]; x < v.obs_offsets[v.num_observables]; x++)
            if (v.obs_meas[x] >= v.num_measurements) return kPackObsLeaf;
    }
    return kPackOk;
}

void pack_finish(PackPlan &pp, uint8_t *img) {
    BatchTotals &t = pp.t;
    if (!t.wide_prob) {
        pp.dict.values(pp.prob_table);
        t.prob_table_n = (uint32_t)pp.prob_table.size();  // (the layout keeps its reserve)
    }
    const StageLayout &L = pp.L;
    auto *lay_noise = (uint32_t *)(img + L.lay_noise);
    auto *lay_meas = (uint32_t *)(img + L.lay_meas);
    auto *lay_src = (uint32_t *)(img + L.lay_src);
    t.sources = 0;
    for (CircuitMeta &m : pp.metas) {  // O(total layers): exclusive prefixes per circuit
        uint32_t meas = 0, src = 0, max_noise = 0, max_meas = 0;
        for (uint32_t i = 0; i <= m.l; i++) {
            const uint32_t li = m.layer_base + i;
            const uint32_t cm = lay_meas[li], cs_ = lay_src[li];
            max_meas = std::max(max_meas, cm);
            if (i < m.l) max_noise = std::max(max_noise, lay_noise[li + 1] - lay_noise[li]);
            lay_meas[li] = meas;
            lay_src[li] = src;
            meas += cm;
            src += cs_;
        }
        m.src_noise = src;
        m.max_layer_noise = max_noise;
        m.src_base = t.sources;
        t.sources += (uint64_t)src + m.M;
        t.max_layer_noise = std::max(t.max_layer_noise, max_noise);
        t.max_layer_meas = std::max(t.max_layer_meas, max_meas);
    }
}

void pack_head(const PackPlan &pp, uint32_t T, uint8_t *img) {
    const BatchTotals &t = pp.t;
    const StageLayout &L = pp.L;
    auto at = [&](uint64_t off) { return img + off; };
    if (!pp.prob_table.empty()) std::memcpy(at(L.prob_table), pp.prob_table.data(), pp.prob_table.size() * 8);
    std::memcpy(at(L.meta), pp.metas.data(), t.C * sizeof(CircuitMeta));
    auto *circ_layer = (uint32_t *)at(L.circ_layer);
    auto *circ_src = (uint64_t *)at(L.circ_src);
    auto *circ_tile = (uint32_t *)at(L.circ_tile);
    auto *circ_grp = (uint32_t *)at(L.circ_grp);
    auto *circ_det = (uint32_t *)at(L.circ_det);
    auto *circ_obs = (uint32_t *)at(L.circ_obs);
    auto *circ_bkt = (uint32_t *)at(L.circ_bkt);
    uint64_t grps = 0, dets = 0, obss = 0;
    for (uint32_t c = 0; c < t.C; c++) {
        const CircuitMeta &m = pp.metas[c];
        circ_layer[c] = (uint32_t)m.circ_layer_base;
        circ_src[c] = m.src_base;
        circ_tile[c] = m.tile_base;
        circ_grp[c] = (uint32_t)grps;
        circ_det[c] = (uint32_t)dets;
        circ_obs[c] = (uint32_t)obss;
        circ_bkt[c] = m.bucket_base;
        grps += (m.W + T - 1) / T;
        dets += m.D;
        obss += m.O;
    }
    circ_layer[t.C] = (uint32_t)t.layers;
    circ_src[t.C] = t.sources;
    circ_tile[t.C] = (uint32_t)t.tiles;
    circ_grp[t.C] = (uint32_t)grps;
    circ_det[t.C] = (uint32_t)dets;
    circ_obs[t.C] = (uint32_t)obss;
    circ_bkt[t.C] = (uint32_t)t.buckets;
}

}  // namespace gp

// gp_gen.cpp -- synthetic workload generators (host, never timed).
//
// gp_gen_repetition / gp_gen_surface restate the reference generators
// (/root/reference/proj/core/src/codes.cpp:149-333, CircuitBuilder
// codes.cpp:23-147) so that the same circuit reaches both compilers; the
// tests pin circuit equality against the reference's own generator.
// gp_gen_bb (bivariate bicycle memory, optional adaptive branch subsets) and
// the SI1000 / uniform noise models are new (the reference has neither;
// SURVEY.md 8d configs 2, 3, 5).
#include <algorithm>
#include <array>
#include <charconv>
#include <cstdlib>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/greenpeas.h"
#include "gp_gen.h"


namespace {

struct Model {
    int kind;  // GP_NOISE_MODEL_*
    double p;
};

// Channel probabilities of a layer (has_mr: the layer holds M / MR / R).
struct ModelProbs {
    double p1, p2, pm, pr, pidle;
};
ModelProbs model_probs(const Model &mdl, bool has_mr) {
    switch (mdl.kind) {
        case GP_NOISE_MODEL_SI1000:
            return {mdl.p / 10, mdl.p, 5 * mdl.p, 2 * mdl.p, has_mr ? 2 * mdl.p : mdl.p / 10};
        case GP_NOISE_MODEL_UNIFORM:
            return {mdl.p, mdl.p, mdl.p, mdl.p, mdl.p};
        default:  // NoiseModel{p}: codes.hpp:30-39
            return {mdl.p, mdl.p / 10, mdl.p, mdl.p, mdl.p / 10};
    }
}

// Open-layer builder (the CircuitBuilder contract: codes.hpp:41-76).
class Builder {
   public:
    explicit Builder(gp_circuit *c) : c_(c) {}
    void h(uint32_t q) { gate(GP_GATE_H, q, 0); }
    void cx(uint32_t a, uint32_t b) { gate(GP_GATE_CX, a, b); }
    void r(uint32_t q) { gate(GP_GATE_R, q, 0); }
    uint32_t m(uint32_t q, double flip = 0) { return meas(GP_GATE_M, q, flip); }
    uint32_t mr(uint32_t q, double flip = 0) { return meas(GP_GATE_MR, q, flip); }
    void noise1(uint8_t kind, double p, uint32_t q) { noise(kind, p, q, 0); }
    void dep2(double p, uint32_t a, uint32_t b) { noise(GP_NOISE_DEPOLARIZE2, p, a, b); }
    void detector(std::vector<uint32_t> ms) {
        std::sort(ms.begin(), ms.end());
        const uint32_t id = (uint32_t)dets_.size();
        dets_.push_back(ms);
        c_->anns.push_back({layer_, false, id, ms});
    }
    void observable_include(uint32_t id, std::vector<uint32_t> ms) {
        std::sort(ms.begin(), ms.end());
        while (obs_.size() <= id) obs_.emplace_back();
        for (uint32_t x : ms) {  // XOR-toggle (codes.cpp:76-92)
            auto &s = obs_[id];
            auto it = std::lower_bound(s.begin(), s.end(), x);
            if (it != s.end() && *it == x) s.erase(it);
            else s.insert(it, x);
        }
        c_->anns.push_back({layer_, true, id, ms});
    }
    void tick() {
        c_->gate_offsets.push_back((uint32_t)c_->gate_kind.size());
        c_->noise_offsets.push_back((uint32_t)c_->noise_kind.size());
        cur_gates_ = cur_noise_ = 0;
        layer_++;
    }
    bool dirty() const {
        bool ann = !c_->anns.empty() && c_->anns.back().layer == layer_;
        return cur_gates_ || cur_noise_ || ann;
    }

    // Decorates the open layer (apply_noise, codes.cpp:94-135 for the paper
    // model): per-gate channels in gate order, then idle channels.
    void apply_noise(const Model &mdl, uint32_t n) {
        std::vector<uint8_t> busy(n, 0);
        const size_t g0 = c_->gate_offsets.back();
        bool has_mr = false;
        for (size_t g = g0; g < c_->gate_kind.size(); g++) {
            uint8_t k = c_->gate_kind[g];
            if (k == GP_GATE_M || k == GP_GATE_MR || k == GP_GATE_R) has_mr = true;
        }
        const ModelProbs mp = model_probs(mdl, has_mr);
        const double p1 = mp.p1, p2 = mp.p2, pm = mp.pm, pr = mp.pr, pidle = mp.pidle;
        for (size_t g = g0; g < c_->gate_kind.size(); g++) {
            const uint32_t q = c_->gate_q0[g];
            busy[q] = 1;
            if (c_->gate_kind[g] == GP_GATE_CX) busy[c_->gate_q1[g]] = 1;
            switch (c_->gate_kind[g]) {
                case GP_GATE_H:
                    if (p1 > 0) noise1(GP_NOISE_DEPOLARIZE1, p1, q);
                    break;
                case GP_GATE_CX:
                    if (p2 > 0) dep2(p2, q, c_->gate_q1[g]);
                    break;
                case GP_GATE_R:
                    if (pr > 0) noise1(GP_NOISE_X_ERROR, pr, q);
                    break;
                case GP_GATE_M:
                    c_->gate_flip[g] = pm;
                    break;
                case GP_GATE_MR:
                    c_->gate_flip[g] = pm;
                    if (pr > 0) noise1(GP_NOISE_X_ERROR, pr, q);
                    break;
            }
        }
        if (pidle > 0)
            for (uint32_t q = 0; q < n; q++)
                if (!busy[q]) noise1(GP_NOISE_DEPOLARIZE1, pidle, q);
    }

    void take(uint32_t n) {
        if (dirty()) tick();
        c_->num_qubits = n;
        c_->num_measurements = meas_count_;
        for (auto &d : dets_) {
            c_->det_meas.insert(c_->det_meas.end(), d.begin(), d.end());
            c_->det_offsets.push_back((uint32_t)c_->det_meas.size());
        }
        for (auto &o : obs_) {
            c_->obs_meas.insert(c_->obs_meas.end(), o.begin(), o.end());
            c_->obs_offsets.push_back((uint32_t)c_->obs_meas.size());
        }
    }
    uint32_t meas_count() const { return meas_count_; }

   private:
    gp_circuit *c_;
    uint32_t layer_ = 0, meas_count_ = 0, cur_gates_ = 0, cur_noise_ = 0;
    std::vector<std::vector<uint32_t>> dets_, obs_;

    void gate(uint8_t k, uint32_t a, uint32_t b) {
        c_->gate_kind.push_back(k);
        c_->gate_q0.push_back(a);
        c_->gate_q1.push_back(b);
        c_->gate_meas.push_back(-1);
        c_->gate_flip.push_back(0);
        cur_gates_++;
    }
    uint32_t meas(uint8_t k, uint32_t q, double flip) {
        gate(k, q, 0);
        c_->gate_meas.back() = (int32_t)meas_count_;
        c_->gate_flip.back() = flip;
        return meas_count_++;
    }
    void noise(uint8_t k, double p, uint32_t a, uint32_t b) {
        c_->noise_kind.push_back(k);
        c_->noise_prob.push_back(p);
        c_->noise_q0.push_back(a);
        c_->noise_q1.push_back(b);
        cur_noise_++;
    }
};

// Rotated surface code layout (surface_layout, codes.cpp:203-243).
struct Check {
    bool is_x;
    uint32_t anc;
    std::vector<uint32_t> support;
    std::array<int32_t, 4> step;
};

std::vector<Check> surface_checks(uint32_t d, uint32_t *nq) {
    static constexpr int kDirs[4][2] = {{-1, -1}, {-1, 0}, {0, -1}, {0, 0}};  // NW NE SW SE
    static constexpr int kStepX[4] = {0, 1, 2, 3};
    static constexpr int kStepZ[4] = {0, 2, 1, 3};
    std::vector<Check> out;
    uint32_t next = d * d;
    for (uint32_t i = 0; i <= d; i++)
        for (uint32_t j = 0; j <= d; j++) {
            const bool is_x = (i + j) % 2 == 1;
            const bool bulk = i >= 1 && i <= d - 1 && j >= 1 && j <= d - 1;
            const bool tb = (i == 0 || i == d) && j >= 1 && j <= d - 1;
            const bool lr = (j == 0 || j == d) && i >= 1 && i <= d - 1;
            if (!(bulk || (tb && is_x) || (lr && !is_x))) continue;
            Check c{is_x, next++, {}, {-1, -1, -1, -1}};
            for (int dir = 0; dir < 4; dir++) {
                const int r = (int)i + kDirs[dir][0], cc = (int)j + kDirs[dir][1];
                if (r < 0 || cc < 0 || r >= (int)d || cc >= (int)d) continue;
                const uint32_t q = (uint32_t)r * d + (uint32_t)cc;
                c.support.push_back(q);
                c.step[is_x ? kStepX[dir] : kStepZ[dir]] = (int32_t)q;
            }
            std::sort(c.support.begin(), c.support.end());
            out.push_back(std::move(c));
        }
    *nq = next;
    return out;
}

// ---- GF(2) helpers for BB logical operators --------------------------------
using Bits = std::vector<uint64_t>;

bool get_bit(const Bits &v, uint32_t i) { return v[i >> 6] >> (i & 63) & 1; }
void xor_into(Bits &a, const Bits &b) {
    for (size_t w = 0; w < a.size(); w++) a[w] ^= b[w];
}

// Incremental echelon basis: reduce(v) eliminates pivots; add(v) inserts.
struct Echelon {
    std::vector<Bits> rows;
    std::vector<uint32_t> piv;
    uint32_t nbits;
    void reduce(Bits &v) const {
        for (size_t r = 0; r < rows.size(); r++)
            if (get_bit(v, piv[r])) xor_into(v, rows[r]);
    }
    bool add(Bits v) {
        reduce(v);
        for (uint32_t i = 0; i < nbits; i++)
            if (get_bit(v, i)) {
                for (auto &r : rows)
                    if (get_bit(r, i)) xor_into(r, v);
                rows.push_back(v);
                piv.push_back(i);
                return true;
            }
        return false;
    }
};

// Null space of H (rows over nbits columns), deterministic basis.
std::vector<Bits> null_space(const std::vector<Bits> &H, uint32_t nbits) {
    Echelon e{{}, {}, nbits};
    for (const Bits &r : H) e.add(r);
    std::vector<uint8_t> is_piv(nbits, 0);
    for (uint32_t p : e.piv) is_piv[p] = 1;
    std::vector<Bits> out;
    const size_t W = (nbits + 63) / 64;
    for (uint32_t f = 0; f < nbits; f++) {
        if (is_piv[f]) continue;
        Bits v(W, 0);
        v[f >> 6] |= 1ull << (f & 63);
        for (size_t r = 0; r < e.rows.size(); r++)  // fully reduced rows: pivot var = row . free part
            if (get_bit(e.rows[r], f)) v[e.piv[r] >> 6] |= 1ull << (e.piv[r] & 63);
        out.push_back(v);
    }
    return out;
}

// Bivariate bicycle geometry (A = x^a0 + y^a1 + y^a2, B = y^b0 + x^b1 + x^b2
// on an L x Mm torus): check k's data qubits per direction, logical Z
// operators. Shared by the host generator (make_bb) and the device branch
// generator's template (bb_template).
struct BBGeom {
    struct Mono {
        uint32_t u, v;
    };
    uint32_t L, Mm, lm, nd, n;
    Mono A[3], B[3];
    BBGeom(uint32_t l, uint32_t m, const uint32_t a[3], const uint32_t b[3])
        : L(l), Mm(m), lm(l * m), nd(2 * l * m), n(4 * l * m),
          A{{a[0], 0}, {0, a[1]}, {0, a[2]}}, B{{0, b[0]}, {b[1], 0}, {b[2], 0}} {}
    uint32_t idx(uint32_t i, uint32_t j) const { return (i % L) * Mm + (j % Mm); }
    uint32_t fwd(Mono mo, uint32_t c) const { return idx(c / Mm + mo.u, c % Mm + mo.v); }
    uint32_t inv(Mono mo, uint32_t c) const { return idx(c / Mm + L - mo.u % L, c % Mm + Mm - mo.v % Mm); }
    // X check c: L data fwd(A_t, c), R data lm + fwd(B_t, c)   (H_X = [A | B])
    // Z check c: L data inv(B_t, c), R data lm + inv(A_t, c)   (H_Z = [B^T | A^T])
    // direction d < 3: the L-data neighbour through A_d (X) or B_d^T (Z);
    // d >= 3: the R-data neighbour through B_{d-3} (X) or A_{d-3}^T (Z)
    uint32_t xdata(int d, uint32_t k) const { return d < 3 ? fwd(A[d], k) : lm + fwd(B[d - 3], k); }
    uint32_t zdata(int d, uint32_t k) const { return d < 3 ? inv(B[d], k) : lm + inv(A[d - 3], k); }
    // Logical Z operators: ker(H_X) modulo rowspace(H_Z).
    std::vector<Bits> logicals() const {
        const size_t W = (nd + 63) / 64;
        std::vector<Bits> HX(lm, Bits(W, 0)), HZ(lm, Bits(W, 0));
        for (uint32_t c = 0; c < lm; c++)
            for (int t = 0; t < 3; t++) {
                uint32_t q;
                q = fwd(A[t], c);
                HX[c][q >> 6] ^= 1ull << (q & 63);
                q = lm + fwd(B[t], c);
                HX[c][q >> 6] ^= 1ull << (q & 63);
                q = inv(B[t], c);
                HZ[c][q >> 6] ^= 1ull << (q & 63);
                q = lm + inv(A[t], c);
                HZ[c][q >> 6] ^= 1ull << (q & 63);
            }
        Echelon span{{}, {}, nd};
        for (const Bits &r : HZ) span.add(r);
        std::vector<Bits> out;
        for (const Bits &v : null_space(HX, nd)) {
            Bits red = v;
            span.reduce(red);
            bool nz = false;
            for (uint64_t w : red) nz |= w != 0;
            if (!nz) continue;
            if (span.add(v)) out.push_back(v);
        }
        return out;
    }
};

// The depth-8 syndrome cycle of Bravyi et al. (Nature 627, 778 (2024),
// Fig. 7): seven CX layers in which X and Z checks interleave, each check
// touching its six data qubits in the direction order kSX / kSZ. Its PrepX /
// MeasX steps are R/MR + H in this gate set, so a round is
//   t0  H(X anc)            | Z: CX dir kSZ[0]
//   t1..t5  X: CX dir kSX[t] | Z: CX dir kSZ[t]
//   t6  X: CX dir kSX[6]     | Z: MR (measure + re-prepare)
//   t7  H(X anc)
//   t8  MR(X anc)
constexpr int kSX[7] = {-1, 1, 4, 3, 5, 0, 2};
constexpr int kSZ[7] = {3, 5, 0, 1, 2, 4, -1};

gp_circuit *make_bb(uint32_t L, uint32_t Mm, const uint32_t a[3], const uint32_t b[3], uint32_t rounds, double p,
                    int model, double check_prob, uint32_t refresh, uint64_t seed, uint64_t branch) {
    const BBGeom geo(L, Mm, a, b);
    const uint32_t lm = geo.lm, nd = geo.nd, n = geo.n;
    auto inv = [&](BBGeom::Mono mo, uint32_t c) { return geo.inv(mo, c); };
    const BBGeom::Mono *A = geo.A, *B = geo.B;
    const std::vector<Bits> logicals = geo.logicals();

    gp_circuit *c = new gp_circuit();
    Builder bld(c);
    const Model mdl{model, p};
    std::seed_seq seq{(uint32_t)seed, (uint32_t)(seed >> 32), (uint32_t)branch, (uint32_t)(branch >> 32)};
    std::mt19937_64 rng(seq);
    std::uniform_real_distribution<double> unif(0.0, 1.0);
    if (refresh == 0) refresh = std::max<uint32_t>(1, rounds / 2);

    for (uint32_t q = 0; q < n; q++) bld.r(q);
    bld.apply_noise(mdl, n);
    bld.tick();
    // Detector tracking (DetectorTracker, adaptive.cpp:114-129): Z checks are
    // deterministic from their first execution, X checks from their second.
    std::vector<int64_t> last_x(lm, -1), last_z(lm, -1);
    for (uint32_t r = 0; r < rounds; r++) {
        const bool full = check_prob >= 1.0 || r == 0 || r + 1 == rounds || r % refresh == 0;
        std::vector<uint8_t> ex(lm, 1), ez(lm, 1);
        if (!full)
            for (uint32_t k = 0; k < lm; k++) {
                ex[k] = unif(rng) < check_prob;
                ez[k] = unif(rng) < check_prob;
            }
        auto xdata = [&](int d, uint32_t k) { return geo.xdata(d, k); };
        auto zdata = [&](int d, uint32_t k) { return geo.zdata(d, k); };
        std::vector<uint32_t> mx(lm), mz(lm);
        for (int t = 0; t < 7; t++) {
            if (t == 0) {
                for (uint32_t k = 0; k < lm; k++)
                    if (ex[k]) bld.h(nd + k);
            } else {
                for (uint32_t k = 0; k < lm; k++)
                    if (ex[k]) bld.cx(nd + k, xdata(kSX[t], k));
            }
            if (t < 6) {
                for (uint32_t k = 0; k < lm; k++)
                    if (ez[k]) bld.cx(zdata(kSZ[t], k), nd + lm + k);
            } else {
                for (uint32_t k = 0; k < lm; k++)
                    if (ez[k]) mz[k] = bld.mr(nd + lm + k);
            }
            bld.apply_noise(mdl, n);
            if (t < 6) bld.tick();
        }
        for (uint32_t k = 0; k < lm; k++)
            if (ez[k]) {
                if (last_z[k] < 0) bld.detector({mz[k]});
                else bld.detector({(uint32_t)last_z[k], mz[k]});
                last_z[k] = mz[k];
            }
        bld.tick();
        for (uint32_t k = 0; k < lm; k++)
            if (ex[k]) bld.h(nd + k);
        bld.apply_noise(mdl, n);
        bld.tick();
        for (uint32_t k = 0; k < lm; k++)
            if (ex[k]) mx[k] = bld.mr(nd + k);
        bld.apply_noise(mdl, n);
        for (uint32_t k = 0; k < lm; k++)
            if (ex[k]) {
                if (last_x[k] >= 0) bld.detector({(uint32_t)last_x[k], mx[k]});
                last_x[k] = mx[k];
            }
        bld.tick();
    }
    std::vector<uint32_t> dm(nd);
    for (uint32_t q = 0; q < nd; q++) dm[q] = bld.m(q);
    bld.apply_noise(mdl, n);
    for (uint32_t k = 0; k < lm; k++) {
        std::vector<uint32_t> set{(uint32_t)last_z[k]};
        for (int t = 0; t < 3; t++) {
            set.push_back(dm[inv(B[t], k)]);
            set.push_back(dm[lm + inv(A[t], k)]);
        }
        bld.detector(set);
    }
    for (uint32_t o = 0; o < logicals.size(); o++) {
        std::vector<uint32_t> set;
        for (uint32_t q = 0; q < nd; q++)
            if (get_bit(logicals[o], q)) set.push_back(dm[q]);
        bld.observable_include(o, set);
    }
    bld.take(n);
    return c;
}

}  // namespace

namespace gp {

const char *bb_template(const gp_bb_spec &s, BBTemplate *t) {
    if (s.l < 2 || s.m < 2 || s.rounds < 1) return "BB spec: l, m >= 2 and rounds >= 1 required";
    const BBGeom geo(s.l, s.m, s.a, s.b);
    t->lm = geo.lm;
    t->nd = geo.nd;
    t->n = geo.n;
    t->rounds = s.rounds;
    t->refresh = s.refresh ? s.refresh : std::max<uint32_t>(1, s.rounds / 2);  // (as make_bb)
    t->check_prob = s.check_prob;
    t->seed = s.seed;
    const Model mdl{s.noise_model, s.p};
    const ModelProbs a = model_probs(mdl, false), b = model_probs(mdl, true);
    t->p1 = a.p1;
    t->p2 = a.p2;
    t->pm = a.pm;
    t->pr = a.pr;
    t->pidle = a.pidle;
    t->pidle_mr = b.pidle;
    const uint32_t lm = geo.lm;
    t->xdata.assign(7 * lm, 0);
    t->zdata.assign(7 * lm, 0);
    for (int x = 0; x < 7; x++)
        for (uint32_t k = 0; k < lm; k++) {
            if (kSX[x] >= 0) t->xdata[x * lm + k] = geo.xdata(kSX[x], k);
            if (kSZ[x] >= 0) t->zdata[x * lm + k] = geo.zdata(kSZ[x], k);
        }
    // Every layer of a full round touches each qubit at most once, so any
    // check subset does too (the device generator counts busy qubits by
    // formula; the reference's validate_layers would reject a collision).
    for (int x = 0; x < 7; x++) {
        std::vector<uint8_t> used(geo.n, 0);
        auto use = [&](uint32_t q) { return used[q]++ == 0; };
        for (uint32_t k = 0; k < lm; k++) {
            bool ok = use(geo.nd + k);
            if (kSX[x] >= 0) ok &= use(t->xdata[x * lm + k]);
            if (kSZ[x] >= 0) ok &= use(t->zdata[x * lm + k]);
            ok &= use(geo.nd + lm + k);
            if (!ok) return "BB spec: a syndrome-cycle layer touches a qubit twice";
        }
    }
    t->zfinal.assign(6 * lm, 0);
    for (uint32_t k = 0; k < lm; k++) {
        uint32_t *z = &t->zfinal[6 * k];
        for (int x = 0; x < 3; x++) {
            z[2 * x] = geo.inv(geo.B[x], k);
            z[2 * x + 1] = lm + geo.inv(geo.A[x], k);
        }
        std::sort(z, z + 6);
        if (std::adjacent_find(z, z + 6) != z + 6) return "BB spec: a final Z detector repeats a data qubit";
    }
    t->obs_off.assign(1, 0);
    t->obs_q.clear();
    for (const Bits &v : geo.logicals()) {
        for (uint32_t q = 0; q < geo.nd; q++)
            if (get_bit(v, q)) t->obs_q.push_back(q);
        t->obs_off.push_back((uint32_t)t->obs_q.size());
    }
    t->O = (uint32_t)t->obs_off.size() - 1;
    return nullptr;
}

}  // namespace gp

extern "C" {

gp_circuit *gp_gen_repetition(uint32_t d, uint32_t rounds, double p) {
    // gen_repetition, codes.cpp:149-201
    if (d < 2 || rounds < 1) return nullptr;
    const uint32_t n = 2 * d - 1, na = d - 1;
    const Model mdl{GP_NOISE_MODEL_PAPER, p};
    gp_circuit *c = new gp_circuit();
    Builder b(c);
    for (uint32_t q = 0; q < n; q++) b.r(q);
    b.apply_noise(mdl, n);
    b.tick();
    std::vector<uint32_t> prev(na), cur(na);
    for (uint32_t r = 0; r < rounds; r++) {
        for (uint32_t a = 0; a < na; a++) b.cx(2 * a, 2 * a + 1);
        b.apply_noise(mdl, n);
        b.tick();
        for (uint32_t a = 0; a < na; a++) b.cx(2 * a + 2, 2 * a + 1);
        b.apply_noise(mdl, n);
        b.tick();
        for (uint32_t a = 0; a < na; a++) cur[a] = b.mr(2 * a + 1);
        b.apply_noise(mdl, n);
        for (uint32_t a = 0; a < na; a++) {
            if (r == 0) b.detector({cur[a]});
            else b.detector({prev[a], cur[a]});
        }
        b.tick();
        prev = cur;
    }
    std::vector<uint32_t> dm(d);
    for (uint32_t i = 0; i < d; i++) dm[i] = b.m(2 * i);
    b.apply_noise(mdl, n);
    for (uint32_t a = 0; a < na; a++) b.detector({prev[a], dm[a], dm[a + 1]});
    b.observable_include(0, {dm[0]});
    b.take(n);
    return c;
}

gp_circuit *gp_gen_surface(uint32_t d, uint32_t rounds, double p, int noise_model, int only_z) {
    // gen_surface, codes.cpp:245-333 (noise_model PAPER reproduces it exactly)
    if (d < 2 || rounds < 1) return nullptr;
    uint32_t n = 0;
    const std::vector<Check> checks = surface_checks(d, &n);
    const Model mdl{noise_model, p};
    gp_circuit *c = new gp_circuit();
    Builder b(c);
    for (uint32_t q = 0; q < n; q++) b.r(q);
    b.apply_noise(mdl, n);
    b.tick();
    std::vector<uint32_t> prev(checks.size()), cur(checks.size());
    for (uint32_t r = 0; r < rounds; r++) {
        for (const Check &k : checks)
            if (k.is_x) b.h(k.anc);
        b.apply_noise(mdl, n);
        b.tick();
        for (int s = 0; s < 4; s++) {
            for (const Check &k : checks) {
                const int32_t q = k.step[s];
                if (q < 0) continue;
                if (k.is_x) b.cx(k.anc, (uint32_t)q);
                else b.cx((uint32_t)q, k.anc);
            }
            b.apply_noise(mdl, n);
            b.tick();
        }
        for (const Check &k : checks)
            if (k.is_x) b.h(k.anc);
        b.apply_noise(mdl, n);
        b.tick();
        for (size_t i = 0; i < checks.size(); i++) cur[i] = b.mr(checks[i].anc);
        b.apply_noise(mdl, n);
        for (size_t i = 0; i < checks.size(); i++) {
            const bool emit = checks[i].is_x ? (!only_z && r > 0) : true;
            if (!emit) continue;
            if (r == 0) b.detector({cur[i]});
            else b.detector({prev[i], cur[i]});
        }
        b.tick();
        prev = cur;
    }
    std::vector<uint32_t> dm(d * d);
    for (uint32_t q = 0; q < d * d; q++) dm[q] = b.m(q);
    b.apply_noise(mdl, n);
    for (size_t i = 0; i < checks.size(); i++) {
        if (checks[i].is_x) continue;
        std::vector<uint32_t> set{prev[i]};
        for (uint32_t q : checks[i].support) set.push_back(dm[q]);
        b.detector(set);
    }
    std::vector<uint32_t> obs;
    for (uint32_t col = 0; col < d; col++) obs.push_back(dm[col]);
    b.observable_include(0, obs);
    b.take(n);
    return c;
}

gp_circuit *gp_gen_bb(uint32_t l, uint32_t m, const uint32_t a[3], const uint32_t b[3], uint32_t rounds, double p,
                      int noise_model, double check_prob, uint32_t refresh, uint64_t seed, uint64_t branch) {
    if (l < 2 || m < 2 || rounds < 1) return nullptr;
    try {
        return make_bb(l, m, a, b, rounds, p, noise_model, check_prob, refresh, seed, branch);
    } catch (...) {
        return nullptr;
    }
}

void gp_circuit_free(gp_circuit *c) { delete c; }

const gp_annotation_view *gp_circuit_annotations(const gp_circuit *c, size_t *count) {
    auto &v = const_cast<gp_circuit *>(c)->ann_views;
    v.clear();
    for (const auto &a : c->anns)
        v.push_back({a.layer, a.is_obs ? 1u : 0u, a.id, (uint32_t)a.meas.size(), a.meas.data()});
    if (count) *count = v.size();
    return v.data();
}

gp_circuit_view gp_circuit_get_view(const gp_circuit *c) {
    gp_circuit_view v{};
    v.num_qubits = c->num_qubits;
    v.num_layers = c->layers();
    v.num_measurements = c->num_measurements;
    v.num_detectors = (uint32_t)c->det_offsets.size() - 1;
    v.num_observables = (uint32_t)c->obs_offsets.size() - 1;
    v.gate_offsets = c->gate_offsets.data();
    v.gate_kind = c->gate_kind.data();
    v.gate_q0 = c->gate_q0.data();
    v.gate_q1 = c->gate_q1.data();
    v.gate_meas = c->gate_meas.data();
    v.gate_flip = c->gate_flip.data();
    v.noise_offsets = c->noise_offsets.data();
    v.noise_kind = c->noise_kind.data();
    v.noise_prob = c->noise_prob.data();
    v.noise_q0 = c->noise_q0.data();
    v.noise_q1 = c->noise_q1.data();
    v.det_offsets = c->det_offsets.data();
    v.det_meas = c->det_meas.data();
    v.obs_offsets = c->obs_offsets.data();
    v.obs_meas = c->obs_meas.data();
    return v;
}

char *gp_circuit_serialize(const gp_circuit *c, size_t *len) {
    // serialize_circuit layout (circuit.cpp:328-388): gates, noise, then the
    // layer's annotations with rec[-k] against the running measurement count.
    std::string s;
    char buf[64];
    auto num = [&](double v) {
        auto r = std::to_chars(buf, buf + sizeof buf, v);
        s.append(buf, r.ptr);
    };
    static const char *kNoise[4] = {"X_ERROR", "Z_ERROR", "DEPOLARIZE1", "DEPOLARIZE2"};
    uint32_t meas = 0;
    size_t ann = 0;
    for (uint32_t i = 0; i < c->layers(); i++) {
        if (i) s += "TICK\n";
        for (uint32_t g = c->gate_offsets[i]; g < c->gate_offsets[i + 1]; g++) {
            switch (c->gate_kind[g]) {
                case GP_GATE_H:
                    s += "H " + std::to_string(c->gate_q0[g]) + "\n";
                    break;
                case GP_GATE_R:
                    s += "R " + std::to_string(c->gate_q0[g]) + "\n";
                    break;
                case GP_GATE_CX:
                    s += "CX " + std::to_string(c->gate_q0[g]) + " " + std::to_string(c->gate_q1[g]) + "\n";
                    break;
                default:
                    s += c->gate_kind[g] == GP_GATE_M ? "M" : "MR";
                    if (c->gate_flip[g] != 0) {
                        s += "(";
                        num(c->gate_flip[g]);
                        s += ")";
                    }
                    s += " " + std::to_string(c->gate_q0[g]) + "\n";
                    meas++;
            }
        }
        for (uint32_t o = c->noise_offsets[i]; o < c->noise_offsets[i + 1]; o++) {
            s += kNoise[c->noise_kind[o]];
            s += "(";
            num(c->noise_prob[o]);
            s += ") " + std::to_string(c->noise_q0[o]);
            if (c->noise_kind[o] == GP_NOISE_DEPOLARIZE2) s += " " + std::to_string(c->noise_q1[o]);
            s += "\n";
        }
        for (; ann < c->anns.size() && c->anns[ann].layer == i; ann++) {
            const auto &a = c->anns[ann];
            s += a.is_obs ? "OBSERVABLE_INCLUDE(" + std::to_string(a.id) + ")" : std::string("DETECTOR");
            for (uint32_t x : a.meas) s += " rec[-" + std::to_string(meas - x) + "]";
            s += "\n";
        }
    }
    char *out = (char *)std::malloc(s.size() + 1);
    std::memcpy(out, s.data(), s.size());
    out[s.size()] = 0;
    if (len) *len = s.size();
    return out;
}

}  // extern "C"

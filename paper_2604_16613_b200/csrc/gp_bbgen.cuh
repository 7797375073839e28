// gp_bbgen.cuh -- branch batches generated on the device (SURVEY.md 8f row
// 3), included by gp_kernels.cu. Seeds in, upload image out: the circuits of
// gp_gen_bb (gp_gen.cpp make_bb) for branch ids first .. first + C - 1 are
// written straight into the staging-image layout the host packer produces
// (gp_pack.cpp), so the unchanged device pipeline compiles them.
//
//   bbgen_draw_kernel  one thread per branch: seed_seq + mt19937_64 (gp_rng.h)
//                      draw the executed check subsets of the non-full rounds
//                      in make_bb's order (per check: X, then Z); per round
//                      masks and counts (the host plans the image from the
//                      counts: gp_gen.h bb_layer_count).
//   bbgen_fill_kernel  one warp per branch: every layer in Builder order --
//                      gates, then per-gate noise channels in gate order, then
//                      idle channels in qubit order (Builder::apply_noise) --
//                      as narrow gate / noise words, measurement flips, layer
//                      tables, detectors (DetectorTracker order) and
//                      observables. Warp ballots place each check's op.

namespace bbgen {

using Params = BBGenParams;

enum : uint32_t { kP1 = 0, kP2 = 1, kPR = 2, kPI = 3, kPIM = 4, kOff = 0xFFFFFFFFu };

__global__ void bbgen_draw_kernel(const Params g) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= g.C) return;
    const uint64_t br = g.first + c;
    uint64_t st[kMtN];
    uint32_t pos = kMtN;
    bool seeded = false;
    for (uint32_t r = 0; r < g.rounds; r++) {
        const bool full = g.check_prob >= 1.0 || r == 0 || r + 1 == g.rounds || r % g.refresh == 0;
        uint64_t *mx = g.masks + ((uint64_t)c * g.rounds + r) * 2 * g.MW, *mz = mx + g.MW;
        uint32_t ne = 0, nz = 0;
        if (full) {
            for (uint32_t w = 0; w < g.MW; w++) {
                const uint32_t bits = min(64u, g.lm - 64 * w);
                mx[w] = mz[w] = bits == 64 ? ~0ull : (1ull << bits) - 1;
            }
            ne = nz = g.lm;
        } else {
            if (!seeded) {  // mt19937_64(seed_seq{seed, seed >> 32, branch, branch >> 32}), make_bb
                const uint32_t s[4] = {(uint32_t)g.seed, (uint32_t)(g.seed >> 32), (uint32_t)br, (uint32_t)(br >> 32)};
                mt64_seed(st, s);
                seeded = true;
            }
            for (uint32_t w = 0; w < g.MW; w++) {
                uint64_t ex = 0, ez = 0;
                for (uint32_t k = 64 * w; k < min(g.lm, 64 * w + 64); k++) {
                    if (mt64_uniform(st, &pos) < g.check_prob) ex |= 1ull << (k & 63);
                    if (mt64_uniform(st, &pos) < g.check_prob) ez |= 1ull << (k & 63);
                }
                mx[w] = ex;
                mz[w] = ez;
                ne += __popcll(ex);
                nz += __popcll(ez);
            }
        }
        g.counts[(uint64_t)c * g.rounds + r] = ne | nz << 16;
    }
}

// Shared memory per warp: busy bitmap (n bits), last Z / X measurement per
// check, this round's Z / X measurement per check.
__host__ __device__ inline uint32_t fill_smem_words(uint32_t n, uint32_t lm) { return (n + 31) / 32 + 4 * lm; }

__global__ void bbgen_fill_kernel(const Params g) {
    extern __shared__ uint32_t sm[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, lt = (1u << lane) - 1;
    const uint32_t c = blockIdx.x * (blockDim.x >> 5) + warp;
    if (c >= g.C) return;
    const uint32_t nw = (g.n + 31) / 32, lm = g.lm;
    uint32_t *busy = sm + warp * fill_smem_words(g.n, lm);
    uint32_t *last_z = busy + nw, *last_x = last_z + lm, *mzv = last_x + lm, *mxv = mzv + lm;
    const StageLayout &L = g.L;
    uint8_t *img = g.img;
    const CircuitMeta m = reinterpret_cast<const CircuitMeta *>(img + L.meta)[c];
    uint32_t *lay_gate = reinterpret_cast<uint32_t *>(img + L.lay_gate) + m.layer_base;
    uint32_t *lay_noise = reinterpret_cast<uint32_t *>(img + L.lay_noise) + m.layer_base;
    uint32_t *lay_meas = reinterpret_cast<uint32_t *>(img + L.lay_meas) + m.layer_base;
    uint32_t *lay_src = reinterpret_cast<uint32_t *>(img + L.lay_src) + m.layer_base;
    uint32_t *gates = reinterpret_cast<uint32_t *>(img + L.gates) + m.gate_base;
    uint32_t *noise = reinterpret_cast<uint32_t *>(img + L.noise) + m.noise_base;
    double *flip = reinterpret_cast<double *>(img + L.meas_flip) + m.meas_base;
    uint32_t *det_off = reinterpret_cast<uint32_t *>(img + L.det_off) + m.det_base;
    uint32_t *det_meas = reinterpret_cast<uint32_t *>(img + L.det_meas) + m.det_entry_base;
    uint32_t *obs_off = reinterpret_cast<uint32_t *>(img + L.obs_off) + m.obs_base;
    uint32_t *obs_meas = reinterpret_cast<uint32_t *>(img + L.obs_meas) + m.obs_entry_base;
    const uint32_t c1 = g.level ? 3 : 2, c2 = g.level == 0 ? 6 : g.level == 1 ? 10 : 15;

    for (uint32_t x = lane; x < lm; x += 32) last_z[x] = last_x[x] = kOff;
    uint32_t ng = 0, nn = 0, ms = 0, src = 0, d = 0, de = 0, li = 0;

    auto begin_layer = [&]() {
        if (lane == 0) {
            lay_gate[li] = (uint32_t)(m.gate_base + ng);
            lay_noise[li] = (uint32_t)(m.noise_base + nn);
            lay_meas[li] = ms;
            lay_src[li] = src;
        }
        for (uint32_t x = lane; x < nw; x += 32) busy[x] = 0;
        __syncwarp();
    };
    // Gates k of [0, N) with sel(k), in k order; each gets its noise channel
    // (ch: kOff for none) right after the previous gates' channels.
    auto segment = [&](uint32_t N, auto sel, auto qubits, uint32_t kind, uint32_t nkind, uint32_t ch, uint32_t *mrec) {
        const uint32_t pi = ch == kOff ? kOff : g.pi[ch];
        const bool meas = kind == GP_GATE_M || kind == GP_GATE_MR;
        for (uint32_t k0 = 0; k0 < N; k0 += 32) {
            const uint32_t k = k0 + lane;
            const bool act = k < N && sel(k);
            const uint32_t bal = __ballot_sync(0xffffffffu, act), pos = __popc(bal & lt);
            if (act) {
                uint32_t q0, q1;
                qubits(k, q0, q1);
                uint32_t hi = kind == GP_GATE_CX ? q1 : 0;
                if (meas) {
                    hi = ms + pos;
                    flip[hi] = g.pm;
                    if (mrec) mrec[k] = hi;
                }
                gates[ng + pos] = narrow_gate(q0, kind, hi);
                atomicOr(&busy[q0 >> 5], 1u << (q0 & 31));
                if (kind == GP_GATE_CX) atomicOr(&busy[q1 >> 5], 1u << (q1 & 31));
                if (pi != kOff) noise[nn + pos] = narrow_noise(q0, nkind == GP_NOISE_DEPOLARIZE2 ? q1 : 0, nkind, pi);
            }
            const uint32_t cnt = __popc(bal);
            ng += cnt;
            if (meas) ms += cnt;
            if (pi != kOff) {
                nn += cnt;
                src += cnt * (nkind == GP_NOISE_DEPOLARIZE2 ? c2 : nkind == GP_NOISE_DEPOLARIZE1 ? c1 : 1);
            }
        }
        __syncwarp();
    };
    auto idle = [&](uint32_t ch) {  // DEPOLARIZE1 on every qubit no gate of the layer touched
        const uint32_t pi = g.pi[ch];
        if (pi == kOff) return;
        for (uint32_t q0 = 0; q0 < g.n; q0 += 32) {
            const uint32_t q = q0 + lane;
            const bool act = q < g.n && !((busy[q >> 5] >> (q & 31)) & 1);
            const uint32_t bal = __ballot_sync(0xffffffffu, act);
            if (act) noise[nn + __popc(bal & lt)] = narrow_noise(q, 0, GP_NOISE_DEPOLARIZE1, pi);
            nn += __popc(bal);
            src += __popc(bal) * c1;
        }
    };
    // Detectors {last[k], cur[k]} (or {cur[k]} without a last) for checks k
    // with sel(k) (DetectorTracker::record, adaptive.cpp:114-129); `need_last`:
    // checks without a previous measurement emit nothing (X checks).
    auto tracker = [&](auto sel, uint32_t *last, const uint32_t *cur, bool need_last) {
        for (uint32_t k0 = 0; k0 < lm; k0 += 32) {
            const uint32_t k = k0 + lane;
            const bool on = k < lm && sel(k);
            const bool has = on && last[k] != kOff;
            const bool act = on && (has || !need_last);
            const uint32_t ent = act ? (has ? 2u : 1u) : 0u;
            uint32_t incl = ent;
#pragma unroll
            for (int s = 1; s < 32; s <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, incl, s);
                if (lane >= (uint32_t)s) incl += o;
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, act);
            if (act) {
                uint32_t e0 = de + incl - ent;
                det_off[d + __popc(bal & lt)] = (uint32_t)(m.det_entry_base + e0);
                if (has) det_meas[e0++] = last[k];
                det_meas[e0] = cur[k];
            }
            if (on) last[k] = cur[k];
            d += __popc(bal);
            de += __shfl_sync(0xffffffffu, incl, 31);
        }
        __syncwarp();
    };

    const uint32_t n = g.n, nd = g.nd;
    auto all = [](uint32_t) { return true; };
    // layer 0: R on every qubit
    begin_layer();
    segment(n, all, [](uint32_t k, uint32_t &q0, uint32_t &q1) { q0 = k, q1 = 0; }, GP_GATE_R, GP_NOISE_X_ERROR, kPR,
            nullptr);
    idle(kPIM);
    li++;
    for (uint32_t r = 0; r < g.rounds; r++) {
        const uint64_t *mx = g.masks + ((uint64_t)c * g.rounds + r) * 2 * g.MW, *mz = mx + g.MW;
        auto ex = [&](uint32_t k) { return (mx[k >> 6] >> (k & 63)) & 1; };
        auto ez = [&](uint32_t k) { return (mz[k >> 6] >> (k & 63)) & 1; };
        const uint32_t cnt = g.counts[(uint64_t)c * g.rounds + r], ne = cnt & 0xFFFF, nz = cnt >> 16;
        for (uint32_t t = 0; t < 7; t++) {
            begin_layer();
            if (t == 0)
                segment(lm, ex, [&](uint32_t k, uint32_t &q0, uint32_t &q1) { q0 = nd + k, q1 = 0; }, GP_GATE_H,
                        GP_NOISE_DEPOLARIZE1, kP1, nullptr);
            else
                segment(lm, ex, [&](uint32_t k, uint32_t &q0, uint32_t &q1) { q0 = nd + k, q1 = g.xdata[t * lm + k]; },
                        GP_GATE_CX, GP_NOISE_DEPOLARIZE2, kP2, nullptr);
            if (t < 6)
                segment(lm, ez,
                        [&](uint32_t k, uint32_t &q0, uint32_t &q1) { q0 = g.zdata[t * lm + k], q1 = nd + lm + k; },
                        GP_GATE_CX, GP_NOISE_DEPOLARIZE2, kP2, nullptr);
            else
                segment(lm, ez, [&](uint32_t k, uint32_t &q0, uint32_t &q1) { q0 = nd + lm + k, q1 = 0; }, GP_GATE_MR,
                        GP_NOISE_X_ERROR, kPR, mzv);
            idle(t == 6 && nz > 0 ? kPIM : kPI);
            if (t == 6) tracker(ez, last_z, mzv, false);
            li++;
        }
        begin_layer();  // H (X anc)
        segment(lm, ex, [&](uint32_t k, uint32_t &q0, uint32_t &q1) { q0 = nd + k, q1 = 0; }, GP_GATE_H,
                GP_NOISE_DEPOLARIZE1, kP1, nullptr);
        idle(kPI);
        li++;
        begin_layer();  // MR (X anc)
        segment(lm, ex, [&](uint32_t k, uint32_t &q0, uint32_t &q1) { q0 = nd + k, q1 = 0; }, GP_GATE_MR,
                GP_NOISE_X_ERROR, kPR, mxv);
        idle(ne > 0 ? kPIM : kPI);
        tracker(ex, last_x, mxv, true);
        li++;
    }
    // final layer: M on the data qubits; Z detectors against the data; observables
    begin_layer();
    const uint32_t M0 = ms;
    segment(nd, all, [](uint32_t k, uint32_t &q0, uint32_t &q1) { q0 = k, q1 = 0; }, GP_GATE_M, 0, kOff, nullptr);
    idle(kPIM);
    for (uint32_t k = lane; k < lm; k += 32) {
        const uint32_t e0 = de + 7 * k;
        det_off[d + k] = (uint32_t)(m.det_entry_base + e0);
        det_meas[e0] = last_z[k];
        for (int j = 0; j < 6; j++) det_meas[e0 + 1 + j] = M0 + g.zfinal[6 * k + j];
    }
    d += lm;
    de += 7 * lm;
    for (uint32_t o = lane; o <= g.O; o += 32) obs_off[o] = (uint32_t)(m.obs_entry_base + g.obs_off[o]);
    for (uint32_t x = lane; x < g.obs_off[g.O]; x += 32) obs_meas[x] = M0 + g.obs_q[x];
    li++;
    if (lane == 0) {  // closing entries; the plan check
        lay_gate[li] = (uint32_t)(m.gate_base + ng);
        lay_noise[li] = (uint32_t)(m.noise_base + nn);
        lay_meas[li] = ms;
        lay_src[li] = src;
        det_off[d] = (uint32_t)(m.det_entry_base + de);
        const CircuitMeta *next = c + 1 < g.C ? reinterpret_cast<const CircuitMeta *>(img + L.meta) + c + 1 : nullptr;
        const uint64_t g_end = next ? next->gate_base : g.gates, n_end = next ? next->noise_base : g.noise;
        const uint64_t de_end = next ? next->det_entry_base : ~0ull;
        if (li != m.l || ms != m.M || d != m.D || src != m.src_noise || m.gate_base + ng != g_end ||
            m.noise_base + nn != n_end || (next && m.det_entry_base + de != de_end))
            atomicAdd(g.err, 1u);
    }
}

}  // namespace bbgen

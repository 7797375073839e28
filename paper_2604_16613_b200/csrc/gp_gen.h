// gp_gen.h -- host side of the device branch generator: the branch-independent
// template of a BB branch batch (gp_gen.cpp bb_template), the per-branch
// layer counts shared by the host planner and the device fill kernel
// (gp_bbgen.cuh), so both agree on every offset.
#pragma once
#include <stdint.h>

#include <vector>

#include "../../include/greenpeas.h"
#include "gp_layout.h"  // (__host__ / __device__ for host-only compiles)

// Owning flat circuit (include/greenpeas.h gp_circuit): the generators' and
// the native parser's output.
struct gp_circuit {
    uint32_t num_qubits = 0, num_measurements = 0;
    std::vector<uint32_t> gate_offsets{0}, noise_offsets{0};
    std::vector<uint8_t> gate_kind, noise_kind;
    std::vector<uint32_t> gate_q0, gate_q1, noise_q0, noise_q1;
    std::vector<int32_t> gate_meas;
    std::vector<double> gate_flip, noise_prob;
    std::vector<uint32_t> det_offsets{0}, det_meas, obs_offsets{0}, obs_meas;
    // Annotation placement for serialization: (layer, is_obs, id, measurements).
    struct Ann {
        uint32_t layer;
        bool is_obs;
        uint32_t id;
        std::vector<uint32_t> meas;
    };
    std::vector<Ann> anns;
    std::vector<gp_annotation_view> ann_views;  // (gp_circuit_annotations)
    uint32_t layers() const { return (uint32_t)gate_offsets.size() - 1; }
};

namespace gp {

struct BBTemplate {
    uint32_t lm = 0, nd = 0, n = 0, rounds = 0, refresh = 0, O = 0;
    double check_prob = 1, p1 = 0, p2 = 0, pm = 0, pr = 0, pidle = 0, pidle_mr = 0;
    uint64_t seed = 0;
    std::vector<uint32_t> xdata;   // [7][lm] layer t: X check k's data qubit (t >= 1)
    std::vector<uint32_t> zdata;   // [7][lm] layer t: Z check k's data qubit (t <= 5)
    std::vector<uint32_t> zfinal;  // [lm][6] data qubits of Z check k's final detector, ascending
    std::vector<uint32_t> obs_off, obs_q;  // logical o: data qubits obs_q[obs_off[o] .. obs_off[o+1]), ascending
};

// nullptr, or why the spec cannot be generated on the device.
const char *bb_template(const gp_bb_spec &s, BBTemplate *t);

// Counts of one layer of a branch circuit (li: 0 = the R layer, 1 + 9 r + t
// = step t of round r (t 0..6 the CX steps, 7 the H step, 8 MR of the X
// ancillas), 1 + 9 R = the final data measurement) given round r's executed
// X / Z checks ne / nz. `on` bits: 1 p1 > 0, 2 p2 > 0, 4 pr > 0, 8 pidle > 0,
// 16 pidle (layers with M / MR / R) > 0 -- Builder::apply_noise (gp_gen.cpp).
struct BBLayerCount {
    uint32_t gates, noise, meas, src;
};
struct BBCountParams {
    uint32_t n, nd, lm, rounds, on, c1, c2;  // c1 / c2: sources per DEPOLARIZE1 / 2 at the level
};
__host__ __device__ inline BBLayerCount bb_layer_count(const BBCountParams &q, uint32_t li, uint32_t ne, uint32_t nz) {
    const bool P1 = q.on & 1, P2 = q.on & 2, PR = q.on & 4, PI = q.on & 8, PIM = q.on & 16;
    auto idle = [&](uint32_t busy, bool has_mr) { return (has_mr ? PIM : PI) ? q.n - busy : 0u; };
    BBLayerCount c{0, 0, 0, 0};
    uint32_t x1 = 0, x2 = 0, xr = 0;  // DEPOLARIZE1, DEPOLARIZE2, X_ERROR ops
    if (li == 0) {  // R on every qubit
        c.gates = q.n;
        xr = PR ? q.n : 0;
    } else if (li == 1 + 9 * q.rounds) {  // M on the data qubits
        c.gates = c.meas = q.nd;
        x1 = idle(q.nd, true);
    } else {
        const uint32_t t = (li - 1) % 9;
        if (t == 0) {  // H (X anc) | CX (Z)
            c.gates = ne + nz;
            x1 = (P1 ? ne : 0) + idle(ne + 2 * nz, false);
            x2 = P2 ? nz : 0;
        } else if (t <= 5) {  // CX | CX
            c.gates = ne + nz;
            x2 = P2 ? ne + nz : 0;
            x1 = idle(2 * ne + 2 * nz, false);
        } else if (t == 6) {  // CX | MR (Z anc)
            c.gates = ne + nz;
            c.meas = nz;
            x2 = P2 ? ne : 0;
            xr = PR ? nz : 0;
            x1 = idle(2 * ne + nz, nz > 0);
        } else if (t == 7) {  // H (X anc)
            c.gates = ne;
            x1 = (P1 ? ne : 0) + idle(ne, false);
        } else {  // MR (X anc)
            c.gates = c.meas = ne;
            xr = PR ? ne : 0;
            x1 = idle(ne, ne > 0);
        }
    }
    c.noise = x1 + x2 + xr;
    c.src = x1 * q.c1 + x2 * q.c2 + xr;
    return c;
}

}  // namespace gp

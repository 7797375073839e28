// demc_shim.cpp -- demc::compile_circuit (include/demc/compile.hpp) over the
// C ABI: demc::Circuit -> flat gp_circuit_view -> gp_compile -> demc::Dem.
// Restores the reference signature (compile.hpp:35-36) and its exception
// behaviour (stepg.cpp:172-174, eec.cpp:44-46 / 52-54).
#include <chrono>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/demc/compile.hpp"
#include "../../include/greenpeas.h"

namespace demc {

namespace {

struct CtxHolder {
    gp_ctx *ctx = nullptr;
    ~CtxHolder() { gp_ctx_destroy(ctx); }
};

// Flattened circuit buffers, reused per host thread.
struct Flat {
    std::vector<uint32_t> gate_off, gate_q0, gate_q1, noise_off, noise_q0, noise_q1, det_off, det_meas, obs_off,
        obs_meas;
    std::vector<uint8_t> gate_kind, noise_kind;
    std::vector<int32_t> gate_meas;
    std::vector<double> gate_flip, noise_prob;
};

gp_ctx *thread_ctx() {
    thread_local CtxHolder h;
    if (!h.ctx) {
        const char *dev = std::getenv("GREENPEAS_DEVICE");
        gp_status st = gp_ctx_create(dev ? std::atoi(dev) : 0, &h.ctx);
        if (st != GP_OK) throw std::runtime_error("greenpeas: no usable CUDA device");
    }
    return h.ctx;
}

gp_circuit_view flatten(const Circuit &c, Flat &f) {
    f = Flat{};
    f.gate_off.push_back(0);
    f.noise_off.push_back(0);
    for (const Layer &L : c.layers) {
        for (const GateOp &g : L.gates) {
            f.gate_kind.push_back((uint8_t)g.kind);
            f.gate_q0.push_back(g.q0);
            f.gate_q1.push_back(g.q1);
            f.gate_meas.push_back(g.meas_index);
            f.gate_flip.push_back(g.flip_prob);
        }
        for (const NoiseOp &n : L.noise) {
            f.noise_kind.push_back((uint8_t)n.kind);
            f.noise_prob.push_back(n.prob);
            f.noise_q0.push_back(n.q0);
            f.noise_q1.push_back(n.q1);
        }
        f.gate_off.push_back((uint32_t)f.gate_kind.size());
        f.noise_off.push_back((uint32_t)f.noise_kind.size());
    }
    f.det_off.push_back(0);
    for (const Detector &d : c.detectors) {
        f.det_meas.insert(f.det_meas.end(), d.measurements.begin(), d.measurements.end());
        f.det_off.push_back((uint32_t)f.det_meas.size());
    }
    f.obs_off.push_back(0);
    for (const Observable &o : c.observables) {
        f.obs_meas.insert(f.obs_meas.end(), o.measurements.begin(), o.measurements.end());
        f.obs_off.push_back((uint32_t)f.obs_meas.size());
    }
    gp_circuit_view v{};
    v.num_qubits = c.num_qubits;
    v.num_layers = (uint32_t)c.layers.size();
    v.num_measurements = c.num_measurements;
    v.num_detectors = (uint32_t)c.detectors.size();
    v.num_observables = (uint32_t)c.observables.size();
    v.gate_offsets = f.gate_off.data();
    v.gate_kind = f.gate_kind.data();
    v.gate_q0 = f.gate_q0.data();
    v.gate_q1 = f.gate_q1.data();
    v.gate_meas = f.gate_meas.data();
    v.gate_flip = f.gate_flip.data();
    v.noise_offsets = f.noise_off.data();
    v.noise_kind = f.noise_kind.data();
    v.noise_prob = f.noise_prob.data();
    v.noise_q0 = f.noise_q0.data();
    v.noise_q1 = f.noise_q1.data();
    v.det_offsets = f.det_off.data();
    v.det_meas = f.det_meas.data();
    v.obs_offsets = f.obs_off.data();
    v.obs_meas = f.obs_meas.data();
    return v;
}

}  // namespace

Dem compile_circuit(const Circuit &c, CorrelationLevel level, uint32_t threads, CompileStats *stats) {
    (void)threads;
    const auto t0 = std::chrono::steady_clock::now();
    thread_local Flat flat;
    gp_ctx *ctx = thread_ctx();
    const gp_circuit_view v = flatten(c, flat);
    gp_dem_view out{};
    gp_stats st{};
    const gp_status rc = gp_compile(ctx, &v, (uint8_t)level, &out, stats ? &st : nullptr);
    if (rc == GP_ERR_INVALID_ARGUMENT) throw std::invalid_argument(gp_last_error(ctx));
    if (rc != GP_OK) throw std::runtime_error(std::string("greenpeas: ") + gp_last_error(ctx));
    Dem d;
    d.num_detectors = out.num_detectors;
    d.num_observables = out.num_observables;
    d.hyperedges.resize(out.num_edges);
    for (uint64_t e = 0; e < out.num_edges; e++) {
        Hyperedge &h = d.hyperedges[e];
        h.detectors.assign(out.det_ids + out.det_offsets[e], out.det_ids + out.det_offsets[e + 1]);
        h.observables.assign(out.obs_ids + out.obs_offsets[e], out.obs_ids + out.obs_offsets[e + 1]);
        h.probability = out.probs[e];
    }
    if (stats) {
        stats->lower_ns = st.lower_ns;
        stats->traverse_ns = st.traverse_ns;
        stats->reduce_ns = st.reduce_ns;
        stats->total_ns = (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                              std::chrono::steady_clock::now() - t0)
                              .count();
    }
    return d;
}

std::string serialize_dem(const Dem &d) {
    // Flatten and reuse the C-ABI formatter (dem.cpp:144-157 semantics).
    std::vector<uint32_t> doff{0}, ooff{0};
    std::vector<uint32_t> dids, oids;
    std::vector<double> probs;
    for (const Hyperedge &h : d.hyperedges) {
        dids.insert(dids.end(), h.detectors.begin(), h.detectors.end());
        oids.insert(oids.end(), h.observables.begin(), h.observables.end());
        doff.push_back((uint32_t)dids.size());
        ooff.push_back((uint32_t)oids.size());
        probs.push_back(h.probability);
    }
    gp_dem_view v{d.num_detectors, d.num_observables, d.hyperedges.size(), doff.data(), dids.data(),
                  ooff.data(),     oids.data(),       probs.data()};
    size_t len = 0;
    char *s = gp_serialize_dem(&v, &len);
    std::string out(s, len);
    gp_free(s);
    return out;
}

}  // namespace demc

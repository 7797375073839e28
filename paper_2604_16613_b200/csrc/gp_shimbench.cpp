// gp_shimbench.cpp -- benchmark harness of the C++ drop-in endpoint
// (libgp_shimbench.so, loaded by bench.py only; not part of the C ABI).
//
// BASELINE.md section 2 asks for two GPU endpoints: the flat pinned DEM
// (gp_compile) and the owning demc::Dem of the reference signature
// (demc::compile_circuit, compile.hpp:35-36, through demc_shim.cpp). This
// times the second one exactly as a reference caller would see it, and the
// reference's own batch pattern over it: T host threads, an atomic work
// counter, one compile_circuit(c, L0, 1) per circuit (demc_main.cpp:184-195).
#include <algorithm>
#include <atomic>
#include <barrier>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "../../include/demc/compile.hpp"
#include "../../include/greenpeas.h"

namespace {

using clk = std::chrono::steady_clock;

demc::Circuit to_circuit(const gp_circuit_view &v) {
    demc::Circuit c;
    c.num_qubits = v.num_qubits;
    c.num_measurements = v.num_measurements;
    c.layers.resize(v.num_layers);
    for (uint32_t i = 0; i < v.num_layers; i++) {
        demc::Layer &L = c.layers[i];
        for (uint32_t g = v.gate_offsets[i]; g < v.gate_offsets[i + 1]; g++)
            L.gates.push_back({(demc::GateKind)v.gate_kind[g], v.gate_q0[g], v.gate_q1[g], v.gate_meas[g],
                               v.gate_flip[g]});
        for (uint32_t o = v.noise_offsets[i]; o < v.noise_offsets[i + 1]; o++)
            L.noise.push_back({(demc::NoiseKind)v.noise_kind[o], v.noise_prob[o], v.noise_q0[o], v.noise_q1[o]});
    }
    for (uint32_t d = 0; d < v.num_detectors; d++)
        c.detectors.push_back({d, std::vector<uint32_t>(v.det_meas + v.det_offsets[d], v.det_meas + v.det_offsets[d + 1])});
    for (uint32_t o = 0; o < v.num_observables; o++)
        c.observables.push_back(
            {o, std::vector<uint32_t>(v.obs_meas + v.obs_offsets[o], v.obs_meas + v.obs_offsets[o + 1])});
    return c;
}

}  // namespace

extern "C" {

// `iters` timed calls of demc::compile_circuit(c, level, 1) after `warmup`
// untimed ones (entry with the circuit in host memory -> owning Dem
// returned); ns_out[iters] receives each call's wall time. Returns the
// hyperedge count, or -1 if a call threw.
int64_t sb_time_shim(const gp_circuit_view *v, int level, uint32_t warmup, uint32_t iters, uint64_t *ns_out) {
    try {
        const demc::Circuit c = to_circuit(*v);
        size_t e = 0;
        for (uint32_t i = 0; i < warmup; i++) e = demc::compile_circuit(c, (demc::CorrelationLevel)level).hyperedges.size();
        for (uint32_t i = 0; i < iters; i++) {
            const auto t0 = clk::now();
            demc::Dem d = demc::compile_circuit(c, (demc::CorrelationLevel)level, 1);
            ns_out[i] = (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(clk::now() - t0).count();
            e = d.hyperedges.size();
        }
        return (int64_t)e;
    } catch (...) {
        return -1;
    }
}

// The demc_main.cpp:184-195 pattern over the drop-in: `threads` persistent
// host threads (each with its own GPU context, sharing the process's packing
// pool) take circuits from an atomic counter, one compile_circuit(c, level, 1)
// each, for `reps` passes over the set; the first pass is untimed (context
// creation, arenas). Returns the hyperedges of one pass; *wall_ns receives the
// mean wall time of a timed pass. -1 on error.
int64_t sb_shim_pool(const gp_circuit_view *views, uint32_t count, int level, uint32_t threads, uint32_t reps,
                     uint64_t *wall_ns) {
    std::vector<demc::Circuit> cs;
    cs.reserve(count);
    for (uint32_t i = 0; i < count; i++) cs.push_back(to_circuit(views[i]));
    reps = std::max<uint32_t>(reps, 2);
    threads = std::max<uint32_t>(threads, 1);
    std::atomic<int64_t> edges{0};
    std::atomic<uint32_t> next{0};
    std::atomic<bool> failed{false};
    std::barrier sync((std::ptrdiff_t)threads + 1);
    std::vector<std::thread> pool;
    for (uint32_t t = 0; t < threads; t++)
        pool.emplace_back([&] {
            for (uint32_t r = 0; r < reps; r++) {
                sync.arrive_and_wait();  // pass r starts
                for (uint32_t s = next++; s < count; s = next++) {
                    try {
                        edges += (int64_t)demc::compile_circuit(cs[s], (demc::CorrelationLevel)level, 1)
                                     .hyperedges.size();
                    } catch (...) {
                        failed = true;
                    }
                }
                sync.arrive_and_wait();  // pass r done
            }
        });
    uint64_t total = 0;
    int64_t one = 0;
    for (uint32_t r = 0; r < reps; r++) {
        next = 0;
        edges = 0;
        sync.arrive_and_wait();
        const auto t0 = clk::now();
        sync.arrive_and_wait();
        if (r) total += (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(clk::now() - t0).count();
        one = edges.load();
    }
    for (auto &th : pool) th.join();
    if (wall_ns) *wall_ns = total / (reps - 1);
    return failed ? -1 : one;
}

// The same pattern for parity: `threads` host threads take circuits from a
// counter, each compile_circuit(c, levels[i], 1) through the drop-in; per
// circuit, status[i] = 0 and digest[i] = gp_dem_digest of the returned
// demc::Dem, or status 1 for std::invalid_argument (its message copied to
// msg[i * 128]), or 2 for any other exception.
int sb_shim_pool_digests(const gp_circuit_view *views, uint32_t count, const uint8_t *levels, uint32_t threads,
                         uint64_t *digest, int32_t *status, char *msg) {
    std::vector<demc::Circuit> cs;
    cs.reserve(count);
    for (uint32_t i = 0; i < count; i++) cs.push_back(to_circuit(views[i]));
    std::atomic<uint32_t> next{0};
    std::vector<std::thread> pool;
    for (uint32_t t = 0; t < std::max<uint32_t>(threads, 1); t++)
        pool.emplace_back([&] {
            for (uint32_t s = next++; s < count; s = next++) {
                try {
                    const demc::Dem d = demc::compile_circuit(cs[s], (demc::CorrelationLevel)levels[s], 1);
                    std::vector<uint32_t> doff{0}, ooff{0}, dids, oids;
                    std::vector<double> pr;
                    for (const auto &h : d.hyperedges) {
                        dids.insert(dids.end(), h.detectors.begin(), h.detectors.end());
                        oids.insert(oids.end(), h.observables.begin(), h.observables.end());
                        doff.push_back((uint32_t)dids.size());
                        ooff.push_back((uint32_t)oids.size());
                        pr.push_back(h.probability);
                    }
                    gp_dem_view v{d.num_detectors, d.num_observables, d.hyperedges.size(), doff.data(),
                                  dids.data(), ooff.data(), oids.data(), pr.data()};
                    digest[s] = gp_dem_digest(&v);
                    status[s] = 0;
                } catch (const std::invalid_argument &e) {
                    status[s] = 1;
                    std::strncpy(msg + (size_t)s * 128, e.what(), 127);
                } catch (...) {
                    status[s] = 2;
                }
            }
        });
    for (auto &th : pool) th.join();
    return 0;
}

}  // extern "C"

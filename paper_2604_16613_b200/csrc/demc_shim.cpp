// demc_shim.cpp -- demc::compile_circuit (include/demc/compile.hpp) over the
// C ABI: demc::Circuit -> flat gp_circuit_view -> gp_compile -> demc::Dem.
// Restores the reference signature (compile.hpp:35-36) and its exception
// behaviour (stepg.cpp:172-174, eec.cpp:44-46 / 52-54).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/demc/circuit.hpp"
#include "../../include/demc/compile.hpp"
#include "../../include/greenpeas.h"

namespace gp {
void host_parallel_for(size_t n, const std::function<void(size_t)> &f);  // gp_api.cpp
void set_compile_overlap(gp_ctx *ctx, std::function<void()> f);           // gp_api.cpp
}

namespace demc {

namespace {

// Work below this many elements stays on the calling thread (a pool wake-up
// costs more than it saves on small circuits).
constexpr size_t kParallelMin = 2048, kGrain = 1024;  // measured: tools/shim_trace.py sweeps
// DEMs from this many hyperedges up have their array built during the compile.
constexpr size_t kPrebuildMin = 4096, kPrebuildMax = 1 << 18;  // (a wrong guess costs at most ~15 MB of zeroing)

// compile_circuit calls in flight in this process: with more than one (host
// threads compiling at once, demc_main.cpp:184-195) the callers already are
// the parallelism and every call stays on its own thread.
std::atomic<int> g_calls{0};
struct CallCount {
    CallCount() { g_calls.fetch_add(1, std::memory_order_relaxed); }
    ~CallCount() { g_calls.fetch_sub(1, std::memory_order_relaxed); }
};

// Contiguous pieces of [0, n) for the pool.
template <class F>
void pieces(size_t n, size_t work, F &&f) {
    static const size_t pmin = std::getenv("GP_SHIM_PAR_MIN") ? std::atol(std::getenv("GP_SHIM_PAR_MIN")) : kParallelMin;
    static const size_t grain = std::getenv("GP_SHIM_GRAIN") ? std::atol(std::getenv("GP_SHIM_GRAIN")) : kGrain;
    const size_t k = work < pmin || g_calls.load(std::memory_order_relaxed) > 1
                         ? 1
                         : std::min<size_t>({64, n, std::max<size_t>(1, work / grain)});
    if (k <= 1) {
        f(0, n);
        return;
    }
    gp::host_parallel_for(k, [&](size_t i) { f(n * i / k, n * (i + 1) / k); });
}

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
    // offsets first (O(layers + detectors)), then the ops and lists copied in
    // parallel pieces
    const size_t L = c.layers.size(), D = c.detectors.size(), O = c.observables.size();
    f.gate_off.resize(L + 1);
    f.noise_off.resize(L + 1);
    f.gate_off[0] = f.noise_off[0] = 0;
    for (size_t i = 0; i < L; i++) {
        f.gate_off[i + 1] = f.gate_off[i] + (uint32_t)c.layers[i].gates.size();
        f.noise_off[i + 1] = f.noise_off[i] + (uint32_t)c.layers[i].noise.size();
    }
    const size_t G = f.gate_off[L], N = f.noise_off[L];
    f.gate_kind.resize(G);
    f.gate_q0.resize(G);
    f.gate_q1.resize(G);
    f.gate_meas.resize(G);
    f.gate_flip.resize(G);
    f.noise_kind.resize(N);
    f.noise_prob.resize(N);
    f.noise_q0.resize(N);
    f.noise_q1.resize(N);
    pieces(L, G + N, [&](size_t a, size_t b) {
        for (size_t i = a; i < b; i++) {
            size_t x = f.gate_off[i];
            for (const GateOp &g : c.layers[i].gates) {
                f.gate_kind[x] = (uint8_t)g.kind;
                f.gate_q0[x] = g.q0;
                f.gate_q1[x] = g.q1;
                f.gate_meas[x] = g.meas_index;
                f.gate_flip[x] = g.flip_prob;
                x++;
            }
            x = f.noise_off[i];
            for (const NoiseOp &n : c.layers[i].noise) {
                f.noise_kind[x] = (uint8_t)n.kind;
                f.noise_prob[x] = n.prob;
                f.noise_q0[x] = n.q0;
                f.noise_q1[x] = n.q1;
                x++;
            }
        }
    });
    f.det_off.resize(D + 1);
    f.det_off[0] = 0;
    for (size_t d = 0; d < D; d++) f.det_off[d + 1] = f.det_off[d] + (uint32_t)c.detectors[d].measurements.size();
    f.det_meas.resize(f.det_off[D]);
    pieces(D, f.det_off[D], [&](size_t a, size_t b) {
        for (size_t d = a; d < b; d++)
            std::copy(c.detectors[d].measurements.begin(), c.detectors[d].measurements.end(),
                      f.det_meas.begin() + f.det_off[d]);
    });
    f.obs_off.assign(1, 0);
    f.obs_meas.clear();
    for (size_t o = 0; o < O; o++) {
        const Observable &ob = c.observables[o];
        f.obs_meas.insert(f.obs_meas.end(), ob.measurements.begin(), ob.measurements.end());
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
    const CallCount in_flight;
    thread_local Flat flat;
    gp_ctx *ctx = thread_ctx();
    const gp_circuit_view v = flatten(c, flat);
    const auto t_flat = std::chrono::steady_clock::now();
    gp_dem_view out{};
    gp_stats st{};
    // The hyperedge array's value-initialisation (56 bytes per edge, one
    // thread) is built while the kernels run, sized like this thread's last
    // DEM, and trimmed or grown to the real size afterwards.
    thread_local size_t last_edges = 0;
    std::vector<Hyperedge> pre;
    const size_t guess = last_edges;
    if (guess >= kPrebuildMin && guess <= kPrebuildMax) gp::set_compile_overlap(ctx, [&pre, guess] { pre.resize(guess); });
    const gp_status rc = gp_compile(ctx, &v, (uint8_t)level, &out, stats ? &st : nullptr);
    gp::set_compile_overlap(ctx, nullptr);
    const auto t_comp = std::chrono::steady_clock::now();
    if (rc == GP_ERR_INVALID_ARGUMENT) throw std::invalid_argument(gp_last_error(ctx));
    if (rc != GP_OK) throw std::runtime_error(std::string("greenpeas: ") + gp_last_error(ctx));
    Dem d;
    d.num_detectors = out.num_detectors;
    d.num_observables = out.num_observables;
    if (2 * out.num_edges >= pre.size()) d.hyperedges = std::move(pre);  // (not for a much smaller DEM: capacity)
    d.hyperedges.resize(out.num_edges);
    last_edges = out.num_edges;
    // one allocation per id list, made on the pool's threads for large DEMs
    // (malloc arenas are per thread)
    pieces(out.num_edges, out.num_edges * 4, [&](size_t a, size_t b) {
        for (size_t e = a; e < b; e++) {
            Hyperedge &h = d.hyperedges[e];
            h.detectors.assign(out.det_ids + out.det_offsets[e], out.det_ids + out.det_offsets[e + 1]);
            h.observables.assign(out.obs_ids + out.obs_offsets[e], out.obs_ids + out.obs_offsets[e + 1]);
            h.probability = out.probs[e];
        }
    });
    static const bool lat = std::getenv("GP_LAT_TRACE") != nullptr;  // experiments: drop-in phase times
    if (lat) {
        const auto ms = [&](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
            return std::chrono::duration<double, std::micro>(b - a).count();
        };
        std::fprintf(stderr, "shim: flatten %.1f  compile %.1f  dem %.1f us\n", ms(t0, t_flat), ms(t_flat, t_comp),
                     ms(t_comp, std::chrono::steady_clock::now()));
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

Circuit parse_circuit(const std::string &text) {
    char *err = nullptr;
    gp_circuit *g = gp_parse_circuit(text.data(), text.size(), &err);
    if (!g) {
        std::string m = err ? err : "parse failed";
        gp_free(err);
        if (m.rfind("line ", 0) == 0) {  // "line N: msg" -> ParseError(N, msg)
            const size_t colon = m.find(": ");
            const size_t line = std::stoul(m.substr(5, colon - 5));
            throw ParseError(line, m.substr(colon + 2));
        }
        throw std::invalid_argument(m);
    }
    const gp_circuit_view v = gp_circuit_get_view(g);
    Circuit c;
    c.num_qubits = v.num_qubits;
    c.num_measurements = v.num_measurements;
    c.layers.resize(v.num_layers);
    for (uint32_t i = 0; i < v.num_layers; i++) {
        Layer &L = c.layers[i];
        for (uint32_t x = v.gate_offsets[i]; x < v.gate_offsets[i + 1]; x++)
            L.gates.push_back({(GateKind)v.gate_kind[x], v.gate_q0[x], v.gate_q1[x], v.gate_meas[x], v.gate_flip[x]});
        for (uint32_t x = v.noise_offsets[i]; x < v.noise_offsets[i + 1]; x++)
            L.noise.push_back({(NoiseKind)v.noise_kind[x], v.noise_prob[x], v.noise_q0[x], v.noise_q1[x]});
    }
    for (uint32_t d = 0; d < v.num_detectors; d++)
        c.detectors.push_back({d, std::vector<uint32_t>(v.det_meas + v.det_offsets[d], v.det_meas + v.det_offsets[d + 1])});
    for (uint32_t o = 0; o < v.num_observables; o++)
        c.observables.push_back({o, std::vector<uint32_t>(v.obs_meas + v.obs_offsets[o], v.obs_meas + v.obs_offsets[o + 1])});
    // annotations, placed in their layers in declaration order
    size_t n = 0;
    const gp_annotation_view *a = gp_circuit_annotations(g, &n);
    for (size_t i = 0; i < n; i++)
        c.layers[a[i].layer].annotations.push_back(
            {a[i].is_observable != 0, a[i].id, std::vector<uint32_t>(a[i].meas, a[i].meas + a[i].num_meas)});
    gp_circuit_free(g);
    return c;
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

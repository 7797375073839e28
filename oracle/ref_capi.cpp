// C ABI over the UNMODIFIED reference library (`demc`), built from the
// reference sources where they lie (/root/reference/proj/core/src/*.cpp) by
// oracle/Makefile into oracle/_ref/libdemc_ref.so.
//
// TEST INFRASTRUCTURE ONLY. This file is glue so that pytest (ctypes) and the
// CPU-baseline leg of bench.py can drive the reference's own public API:
//   parse_circuit        circuit.cpp:107
//   compile_circuit      compile.cpp:23-53   (the hot path being replaced)
//   build_dem_oracle     frame.cpp:200-239   (forward-propagation oracle)
//   serialize_dem        dem.cpp:144-157
//   gen_surface / gen_repetition  codes.cpp:149-333
//   run_adaptive_shot    adaptive.cpp:382-391
// Nothing in the product path (paper_2604_16613_b200/) links or loads this.
//
// Workload circuits the reference has no generator for (BB / SI1000 /
// adaptive branches) come from this repo's host generator
// source (paper_2604_16613_b200/csrc/gp_gen.cpp), compiled INTO this library
// with hidden visibility by oracle/Makefile, and reach the reference only as
// circuit text through its own parse_circuit -- so the --impl reference arm of
// bench.py loads nothing but this library.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "demc/adaptive.hpp"
#include "demc/codes.hpp"
#include "demc/compile.hpp"
#include "demc/frame.hpp"
#include "greenpeas.h"

namespace {

thread_local std::string g_err;

char *dup_string(const std::string &s, size_t *len) {
    char *out = (char *)std::malloc(s.size() + 1);
    std::memcpy(out, s.data(), s.size());
    out[s.size()] = 0;
    if (len) *len = s.size();
    return out;
}

// DEM digest: the same 64-bit hash as gp_dem_digest (include/greenpeas.h),
// restated over the reference's own demc::Dem. Equal digests <=> identical
// serialize_dem text (ids exact, probability bits exact; shortest round-trip
// formatting is injective on doubles).
uint64_t dg_mix(uint64_t h, uint64_t w) {
    uint64_t x = h + w + 0x9e3779b97f4a7c15ull;
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

uint64_t dem_digest(const demc::Dem &d) {
    uint64_t h = 0x6a09e667f3bcc909ull;
    h = dg_mix(h, (uint64_t)d.num_detectors << 32 | d.num_observables);
    h = dg_mix(h, d.hyperedges.size());
    for (const demc::Hyperedge &e : d.hyperedges) {
        h = dg_mix(h, (uint64_t)e.detectors.size() << 32 | e.observables.size());
        for (uint32_t x : e.detectors) h = dg_mix(h, x);
        for (uint32_t x : e.observables) h = dg_mix(h, x);
        uint64_t bits;
        std::memcpy(&bits, &e.probability, 8);
        h = dg_mix(h, bits);
    }
    return h;
}

template <class F>
void parallel_for(uint32_t count, uint32_t threads, F &&f) {
    std::atomic<uint32_t> next{0};
    std::vector<std::thread> pool;
    for (uint32_t t = 0; t < std::max<uint32_t>(1, threads); t++)
        pool.emplace_back([&] {
            for (uint32_t s = next++; s < count; s = next++) f(s);
        });
    for (auto &th : pool) th.join();
}

}  // namespace

extern "C" {

const char *ref_last_error() { return g_err.c_str(); }

void ref_free(void *p) { std::free(p); }

// Parses circuit text and returns an opaque handle (nullptr on error).
void *ref_circuit_parse(const char *text) {
    try {
        return new demc::Circuit(demc::parse_circuit(text));
    } catch (const std::exception &e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_circuit_free(void *h) { delete (demc::Circuit *)h; }

// Serialized circuit text of a handle (reference grammar).
char *ref_circuit_text(void *h, size_t *len) {
    return dup_string(demc::serialize_circuit(*(demc::Circuit *)h), len);
}

// compile_circuit + serialize_dem. Returns malloc'd DEM text or nullptr.
// stats (optional) receives {lower_ns, traverse_ns, reduce_ns, total_ns, E}.
char *ref_compile(void *h, int level, uint32_t threads, uint64_t *stats, size_t *len) {
    try {
        demc::CompileStats st;
        demc::Dem d = demc::compile_circuit(*(demc::Circuit *)h, (demc::CorrelationLevel)level,
                                            threads, &st);
        if (stats) {
            stats[0] = st.lower_ns;
            stats[1] = st.traverse_ns;
            stats[2] = st.reduce_ns;
            stats[3] = st.total_ns;
            stats[4] = d.hyperedges.size();
        }
        return dup_string(demc::serialize_dem(d), len);
    } catch (const std::exception &e) {
        g_err = e.what();
        return nullptr;
    }
}

// Forward-propagation oracle (frame.cpp:200-239), serialized.
char *ref_oracle(void *h, int level, size_t *len) {
    try {
        return dup_string(
            demc::serialize_dem(demc::build_dem_oracle(*(demc::Circuit *)h, (demc::CorrelationLevel)level)),
            len);
    } catch (const std::exception &e) {
        g_err = e.what();
        return nullptr;
    }
}

void *ref_gen_surface(uint32_t d, uint32_t rounds, double p, int only_z) {
    try {
        return new demc::Circuit(demc::gen_surface(d, rounds, demc::NoiseModel{p}, only_z != 0));
    } catch (const std::exception &e) {
        g_err = e.what();
        return nullptr;
    }
}

void *ref_gen_repetition(uint32_t d, uint32_t rounds, double p) {
    try {
        return new demc::Circuit(demc::gen_repetition(d, rounds, demc::NoiseModel{p}));
    } catch (const std::exception &e) {
        g_err = e.what();
        return nullptr;
    }
}

// One adaptive Iceberg shot (adaptive.cpp:382-391): returns the realized
// circuit handle; *dem_text receives the reference DEM of that shot.
void *ref_adaptive_shot(uint32_t d, uint32_t rounds, uint32_t refresh, double p, uint64_t seed,
                        uint64_t shot, char **dem_text, size_t *dem_len) {
    try {
        demc::AdaptiveConfig cfg;
        cfg.d = d;
        cfg.rounds = rounds;
        cfg.refresh = refresh;
        cfg.p = p;
        cfg.seed = seed;
        demc::ShotRecord rec = demc::run_adaptive_shot(cfg, shot);
        if (dem_text) *dem_text = dup_string(demc::serialize_dem(rec.dem), dem_len);
        return new demc::Circuit(std::move(rec.circuit));
    } catch (const std::exception &e) {
        g_err = e.what();
        return nullptr;
    }
}

// Times `iters` calls of compile_circuit(c, level, 1) after one warm-up
// (the demc_main.cpp:126-133 methodology). ns_out[iters] receives each total.
// Returns the hyperedge count, or -1 on error.
int64_t ref_time_compile(void *h, int level, uint32_t iters, uint64_t *ns_out) {
    try {
        const demc::Circuit &c = *(demc::Circuit *)h;
        size_t e = demc::compile_circuit(c, (demc::CorrelationLevel)level, 1).hyperedges.size();
        for (uint32_t i = 0; i < iters; i++) {
            auto t0 = std::chrono::steady_clock::now();
            demc::Dem d = demc::compile_circuit(c, (demc::CorrelationLevel)level, 1);
            auto t1 = std::chrono::steady_clock::now();
            ns_out[i] = (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
            e = d.hyperedges.size();
        }
        return (int64_t)e;
    } catch (const std::exception &e) {
        g_err = e.what();
        return -1;
    }
}

// serialize_dem (dem.cpp:144-157) of the circuit's DEM, `iters` timed calls
// (the compile itself untimed). Returns the text length, -1 on error.
int64_t ref_time_serialize(void *h, int level, uint32_t iters, uint64_t *ns_out) {
    try {
        const demc::Dem d = demc::compile_circuit(*(demc::Circuit *)h, (demc::CorrelationLevel)level, 1);
        size_t n = 0;
        for (uint32_t i = 0; i < iters; i++) {
            auto t0 = std::chrono::steady_clock::now();
            const std::string text = demc::serialize_dem(d);
            auto t1 = std::chrono::steady_clock::now();
            ns_out[i] = (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
            n = text.size();
        }
        return (int64_t)n;
    } catch (const std::exception &e) {
        g_err = e.what();
        return -1;
    }
}

// Compiles `count` circuits on a std::thread pool of `threads` workers with an
// atomic work counter, one compile_circuit(..., 1) per circuit (the
// demc_main.cpp:184-195 pattern). Returns the total hyperedge count; *wall_ns
// receives the wall time of the pool run. -1 on error.
int64_t ref_compile_pool(void **handles, uint32_t count, int level, uint32_t threads,
                         uint64_t *wall_ns) {
    std::atomic<uint32_t> next{0};
    std::atomic<int64_t> total{0};
    std::atomic<bool> failed{false};
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (uint32_t t = 0; t < std::max<uint32_t>(1, threads); t++) {
        pool.emplace_back([&] {
            for (uint32_t s = next++; s < count; s = next++) {
                try {
                    demc::Dem d = demc::compile_circuit(*(demc::Circuit *)handles[s],
                                                        (demc::CorrelationLevel)level, 1);
                    total += (int64_t)d.hyperedges.size();
                } catch (...) {
                    failed = true;
                }
            }
        });
    }
    for (auto &th : pool) th.join();
    auto t1 = std::chrono::steady_clock::now();
    if (wall_ns)
        *wall_ns = (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
    return failed ? -1 : total.load();
}

// BB [[72,12,6]] adaptive branch circuits as
// reference circuits: branch first + i -> handles[i], generated by the repo's
// host generator (gp_gen_bb, hidden in this library) and parsed from text by
// the reference's parse_circuit on `threads` workers. 0 on success.
int ref_gen_bb72_branches(uint64_t first, uint32_t count, uint32_t rounds, double p, double check_prob,
                          uint64_t seed, uint32_t threads, void **handles) {
    static const uint32_t a[3] = {3, 1, 2}, b[3] = {3, 1, 2};
    std::atomic<bool> failed{false};
    parallel_for(count, threads, [&](uint32_t i) {
        handles[i] = nullptr;
        gp_circuit *g = gp_gen_bb(6, 6, a, b, rounds, p, GP_NOISE_MODEL_PAPER, check_prob,
                                  std::max<uint32_t>(1, rounds / 2), seed, first + i);
        if (!g) {
            failed = true;
            return;
        }
        size_t n = 0;
        char *text = gp_circuit_serialize(g, &n);
        gp_circuit_free(g);
        try {
            handles[i] = new demc::Circuit(demc::parse_circuit(std::string(text, n)));
        } catch (...) {
            failed = true;
        }
        std::free(text);
    });
    return failed ? -1 : 0;
}

// compile_circuit(c, level, 1) of every handle on `threads` workers (not
// timed): per circuit, hyperedge count and DEM digest (dem_digest above).
int ref_compile_digests(void **handles, uint32_t count, int level, uint32_t threads, uint64_t *edges,
                        uint64_t *digests) {
    std::atomic<bool> failed{false};
    parallel_for(count, threads, [&](uint32_t s) {
        try {
            demc::Dem d = demc::compile_circuit(*(demc::Circuit *)handles[s], (demc::CorrelationLevel)level, 1);
            edges[s] = d.hyperedges.size();
            digests[s] = dem_digest(d);
        } catch (...) {
            failed = true;
        }
    });
    return failed ? -1 : 0;
}

// Digest of a DEM given as text (parse_dem, dem.cpp:158-197).
uint64_t ref_dem_text_digest(const char *text, uint32_t num_detectors, uint32_t num_observables) {
    return dem_digest(demc::parse_dem(text, num_detectors, num_observables));
}

// Noiseless-soundness probe (frame.cpp:241-248, collapse randomisation on):
// number of (shot, detector) pairs that fired over `shots` shots.
int64_t ref_sample_fired(void *h, uint64_t seed, uint32_t shots) {
    try {
        std::mt19937_64 rng(seed);
        int64_t fired = 0;
        for (uint32_t s = 0; s < shots; s++)
            for (uint8_t v : demc::sample_detector_values(*(demc::Circuit *)h, rng)) fired += v;
        return fired;
    } catch (const std::exception &e) {
        g_err = e.what();
        return -1;
    }
}

}  // extern "C"

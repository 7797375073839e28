// demc/compile.hpp -- the drop-in replacement of the reference hot path
//     Dem compile_circuit(const Circuit &, CorrelationLevel, uint32_t, CompileStats *)
// (reference: core/include/demc/compile.hpp:26-36, core/src/compile.cpp:23-53),
// implemented over the C ABI in greenpeas.h by libgreenpeas.so.
//
// Same contract: the circuit is caller-owned and validated; the result is an
// owning Dem in canonical order; std::invalid_argument carries the
// reference's messages; calls are reentrant (one GPU context per host
// thread). `threads` is accepted for source compatibility; the output does
// not depend on it, exactly as in the reference (compile.hpp:33-34).
// The device is cuda:0 unless GREENPEAS_DEVICE is set.
#ifndef GREENPEAS_DEMC_COMPILE_HPP
#define GREENPEAS_DEMC_COMPILE_HPP

#include <cstdint>

#include "demc/circuit.hpp"
#include "demc/dem.hpp"
#include "demc/stepg.hpp"

namespace demc {

struct CompileStats {
    uint64_t lower_ns = 0;
    uint64_t traverse_ns = 0;
    uint64_t reduce_ns = 0;
    uint64_t total_ns = 0;
};

Dem compile_circuit(const Circuit &c, CorrelationLevel level, uint32_t threads = 1,
                    CompileStats *stats = nullptr);

}  // namespace demc

#endif

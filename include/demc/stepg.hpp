// demc/stepg.hpp -- correlation level of the drop-in boundary
// (reference: core/include/demc/stepg.hpp:28). The STEPG itself is built on
// the GPU (gp_kernels.cu) and is not exposed.
#ifndef GREENPEAS_DEMC_STEPG_HPP
#define GREENPEAS_DEMC_STEPG_HPP

#include <cstdint>

namespace demc {

enum class CorrelationLevel : uint8_t { L0 = 0, L1 = 1, L2 = 2 };  // == GP_LEVEL_*

}  // namespace demc

#endif

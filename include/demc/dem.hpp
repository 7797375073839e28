// demc/dem.hpp -- DEM value types of the drop-in boundary
// (reference: core/include/demc/dem.hpp:28-52, 144-157).
#ifndef GREENPEAS_DEMC_DEM_HPP
#define GREENPEAS_DEMC_DEM_HPP

#include <cstdint>
#include <string>
#include <vector>

namespace demc {

// Probability that exactly one of two independent events fires.
inline double merge_prob(double a, double b) { return a * (1 - b) + b * (1 - a); }

struct Hyperedge {
    std::vector<uint32_t> detectors;    // ascending
    std::vector<uint32_t> observables;  // ascending
    double probability;
    bool operator==(const Hyperedge &) const = default;
};

struct Dem {
    uint32_t num_detectors = 0;
    uint32_t num_observables = 0;
    std::vector<Hyperedge> hyperedges;  // canonical (detectors, observables) order
    bool operator==(const Dem &) const = default;
};

// `error(<shortest round-trip>) D.. L..` per hyperedge.
std::string serialize_dem(const Dem &d);

}  // namespace demc

#endif

/* demc_oracle.h -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain-C restatement of the reference compile path
 * (/root/reference/proj/core/src/{stepg,eec,dem,compile,frame}.cpp) used only
 * by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * CHECKER of the CUDA path. It follows the reference structure literally
 * (alpha = 2/4/7 slots per qubit, correlated slots, dense column-major class
 * matrix, FNV-1 keyed sort/reduce), so agreement with it also validates the
 * product's base-slot shortcut.
 *
 * Parity is pinned: tests/test_oracle.py checks this restatement against the
 * reference's four golden fixtures (proj/fixtures/*, copied to
 * tests/golden/fixtures) and against the reference library itself compiled
 * from its own sources (oracle/_ref/libdemc_ref.so) on generated circuits.
 *
 * Input is the flat circuit layout of include/greenpeas.h (gp_circuit_view),
 * passed as raw arrays so the oracle has no dependency on product code.
 */
#ifndef DEMC_ORACLE_H
#define DEMC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_circuit {
    uint32_t num_qubits, num_layers, num_measurements, num_detectors, num_observables;
    const uint32_t *gate_offsets; /* [num_layers + 1] */
    const uint8_t *gate_kind;     /* 0 H, 1 CX, 2 R, 3 M, 4 MR  (circuit.hpp:35) */
    const uint32_t *gate_q0;
    const uint32_t *gate_q1;
    const int32_t *gate_meas;
    const double *gate_flip;
    const uint32_t *noise_offsets; /* [num_layers + 1] */
    const uint8_t *noise_kind;     /* 0 X_ERROR, 1 Z_ERROR, 2 DEPOLARIZE1, 3 DEPOLARIZE2 */
    const double *noise_prob;
    const uint32_t *noise_q0;
    const uint32_t *noise_q1;
    const uint32_t *det_offsets; /* [num_detectors + 1] */
    const uint32_t *det_meas;
    const uint32_t *obs_offsets; /* [num_observables + 1] */
    const uint32_t *obs_meas;
} oracle_circuit;

/* Flat DEM: hyperedges in canonical order (dem.cpp:122-127). */
typedef struct oracle_dem {
    uint32_t num_detectors, num_observables;
    uint64_t num_edges;
    uint64_t *det_offsets; /* [E + 1] */
    uint32_t *det_ids;
    uint64_t *obs_offsets; /* [E + 1] */
    uint32_t *obs_ids;
    double *probs;          /* [E] */
    uint64_t num_sources;   /* graph-level error sources (stepg.cpp:269-313) */
    uint64_t *mem_offsets;  /* [E + 1] members per hyperedge (dem.cpp:87-121) */
    uint32_t *mem_ids;      /* source indices, ascending within a hyperedge */
} oracle_dem;

/* Returns 0 on success; on failure a nonzero code and a message via
 * oracle_last_error():
 *   1 "circuit exceeds 32-bit node index space"            (stepg.cpp:172-174)
 *   2 "detector references a measurement without a leaf"   (eec.cpp:44-46)
 *   3 "observable references a measurement without a leaf" (eec.cpp:52-54)
 *   4 out of memory */
int oracle_compile(const oracle_circuit *c, int level, oracle_dem *out);

/* Forward-propagation oracle (frame.cpp:159-239): O(S * l * n). */
int oracle_forward(const oracle_circuit *c, int level, oracle_dem *out);

void oracle_dem_free(oracle_dem *d);
const char *oracle_last_error(void);

/* Known-answer helpers (dem.cpp:27-37, dem.hpp:28-30). */
uint64_t oracle_fnv1_64(const uint64_t *words, size_t n);
double oracle_merge_prob(double a, double b);

#ifdef __cplusplus
}
#endif
#endif

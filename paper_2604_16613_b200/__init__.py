"""paper_2604_16613_b200 -- B200-native GreenPeas DEM compiler.

Drop-in for the reference hot path demc::compile_circuit
(/root/reference/proj/core/src/compile.cpp:23-53): circuit in, detector
error model out, computed by sm_100a CUDA kernels (csrc/gp_kernels.cu)
behind the C ABI of include/greenpeas.h.
"""

from .api import (  # noqa: F401
    NOISE_MODEL_PAPER,
    NOISE_MODEL_SI1000,
    NOISE_MODEL_UNIFORM,
    OPT_FORCE_HASH_COLLISIONS,
    OPT_RECORD_SLOTS,
    Compiler,
    CorrelationLevel,
    Dem,
    DevicePartialTable,
    GenCircuit,
    GreenpeasError,
    PartialTable,
    algorithmic_bytes,
    circuit_metrics,
    compile_circuit,
    gen_bb,
    gen_bb72_branch,
    parse_circuit_native,
    CircuitParseError,
    bb_spec,
    bb72_branch_spec,
    gen_bb144,
    gen_repetition,
    gen_surface,
)
from .circuit import Circuit, ParseError, merge_prob, parse_circuit, serialize_circuit, validate_layers  # noqa: F401

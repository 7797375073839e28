"""ctypes binding of libgreenpeas.so (include/greenpeas.h).

The library is built in-tree by paper_2604_16613_b200.build. There is no
fallback: if the shared library is missing or fails to load, importing the
compile API raises.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libgreenpeas.so"

_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_u64p = C.POINTER(C.c_uint64)
_f64p = C.POINTER(C.c_double)


class CircuitView(C.Structure):
    _fields_ = [
        ("num_qubits", C.c_uint32), ("num_layers", C.c_uint32), ("num_measurements", C.c_uint32),
        ("num_detectors", C.c_uint32), ("num_observables", C.c_uint32),
        ("gate_offsets", _u32p), ("gate_kind", _u8p), ("gate_q0", _u32p), ("gate_q1", _u32p),
        ("gate_meas", _i32p), ("gate_flip", _f64p),
        ("noise_offsets", _u32p), ("noise_kind", _u8p), ("noise_prob", _f64p), ("noise_q0", _u32p),
        ("noise_q1", _u32p),
        ("det_offsets", _u32p), ("det_meas", _u32p), ("obs_offsets", _u32p), ("obs_meas", _u32p),
    ]


class DemView(C.Structure):
    _fields_ = [
        ("num_detectors", C.c_uint32), ("num_observables", C.c_uint32), ("num_edges", C.c_uint64),
        ("det_offsets", _u32p), ("det_ids", _u32p), ("obs_offsets", _u32p), ("obs_ids", _u32p),
        ("probs", _f64p),
    ]


class DemBatchView(C.Structure):
    _fields_ = [
        ("num_circuits", C.c_uint64), ("edge_offsets", _u64p), ("num_detectors", _u32p),
        ("num_observables", _u32p), ("num_edges", C.c_uint64),
        ("det_offsets", _u32p), ("det_ids", _u32p), ("obs_offsets", _u32p), ("obs_ids", _u32p),
        ("probs", _f64p),
    ]


class PartialView(C.Structure):
    _fields_ = [
        ("num_detectors", C.c_uint32), ("num_observables", C.c_uint32), ("num_sources", C.c_uint64),
        ("num_records", C.c_uint64), ("memory", C.c_uint32), ("reserved", C.c_uint32), ("probs", _f64p), ("rec_offsets", _u32p), ("rec_words", _u32p),
        ("rec_bits", _u64p),
    ]


class Metrics(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("base_nodes", "succ_refs", "source_rows", "sources", "words",
                                          "measurements")]


class BBSpec(C.Structure):  # gp_bb_spec
    _fields_ = [("l", C.c_uint32), ("m", C.c_uint32), ("a", C.c_uint32 * 3), ("b", C.c_uint32 * 3),
                ("rounds", C.c_uint32), ("refresh", C.c_uint32), ("noise_model", C.c_int32),
                ("reserved", C.c_uint32), ("p", C.c_double), ("check_prob", C.c_double), ("seed", C.c_uint64)]


class Stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "lower_ns", "traverse_ns", "reduce_ns", "total_ns", "h2d_ns", "kernel_ns", "d2h_ns",
        "num_sources", "h2d_bytes", "d2h_bytes", "kernel_launches", "traverse_kernel_ns")]

    def as_dict(self) -> dict:
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2604_16613_b200.build` "
                               "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        vp = C.c_void_p
        L.gp_ctx_create.argtypes = [C.c_int, C.POINTER(vp)]
        L.gp_ctx_destroy.argtypes = [vp]
        L.gp_last_error.argtypes = [vp]
        L.gp_last_error.restype = C.c_char_p
        L.gp_ctx_set_option.argtypes = [vp, C.c_int, C.c_int64]
        L.gp_compile.argtypes = [vp, C.POINTER(CircuitView), C.c_uint8, C.POINTER(DemView), C.POINTER(Stats)]
        L.gp_compile_batch.argtypes = [vp, C.POINTER(CircuitView), C.c_size_t, C.c_uint8,
                                       C.POINTER(DemBatchView), C.POINTER(Stats)]
        L.gp_compile_bb_branches.argtypes = [vp, C.POINTER(BBSpec), C.c_uint64, C.c_size_t, C.c_uint8,
                                             C.POINTER(DemBatchView), C.POINTER(Stats)]
        L.gp_compile_shard.argtypes = [vp, C.POINTER(CircuitView), C.c_uint8, C.c_uint32, C.c_uint32,
                                       C.c_uint32, C.POINTER(PartialView), C.POINTER(Stats)]
        L.gp_merge_partials.argtypes = [vp, C.POINTER(PartialView), C.c_size_t, C.POINTER(DemView),
                                        C.POINTER(Stats)]
        L.gp_replay.argtypes = [vp, C.c_uint32, C.c_int, C.POINTER(Stats)]
        L.gp_profile_stages.argtypes = [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_char_p), C.c_int]
        L.gp_circuit_metrics.argtypes = [C.POINTER(CircuitView), C.c_uint8, C.POINTER(Metrics)]
        L.gp_serialize_dem.argtypes = [C.POINTER(DemView), C.POINTER(C.c_size_t)]
        L.gp_serialize_dem.restype = vp
        L.gp_dem_digest.argtypes = [C.POINTER(DemView)]
        L.gp_dem_digest.restype = C.c_uint64
        L.gp_dem_batch_digest.argtypes = [C.POINTER(DemBatchView), _u64p]
        L.gp_free.argtypes = [vp]
        L.gp_host_alloc.argtypes = [C.c_size_t]
        L.gp_host_alloc.restype = vp
        L.gp_host_free.argtypes = [vp]
        L.gp_gen_repetition.argtypes = [C.c_uint32, C.c_uint32, C.c_double]
        L.gp_gen_repetition.restype = vp
        L.gp_gen_surface.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_int, C.c_int]
        L.gp_gen_surface.restype = vp
        L.gp_gen_bb.argtypes = [C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                C.c_uint32, C.c_double, C.c_int, C.c_double, C.c_uint32, C.c_uint64,
                                C.c_uint64]
        L.gp_gen_bb.restype = vp
        L.gp_circuit_free.argtypes = [vp]
        L.gp_circuit_get_view.argtypes = [vp]
        L.gp_circuit_get_view.restype = CircuitView
        L.gp_parse_circuit.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(C.c_void_p)]
        L.gp_parse_circuit.restype = vp
        L.gp_circuit_serialize.argtypes = [vp, C.POINTER(C.c_size_t)]
        L.gp_circuit_serialize.restype = vp
        _lib = L
    return _lib


def take_string(ptr, n) -> str:
    s = C.string_at(ptr, n).decode()
    lib().gp_free(ptr)
    return s


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def view_of(c) -> tuple[CircuitView, tuple]:
    """gp_circuit_view over a Circuit's numpy arrays (kept alive by the tuple)."""
    arrs = tuple(np.ascontiguousarray(getattr(c, n), dtype=dt) for n, dt in (
        ("gate_offsets", np.uint32), ("gate_kind", np.uint8), ("gate_q0", np.uint32), ("gate_q1", np.uint32),
        ("gate_meas", np.int32), ("gate_flip", np.float64), ("noise_offsets", np.uint32),
        ("noise_kind", np.uint8), ("noise_prob", np.float64), ("noise_q0", np.uint32), ("noise_q1", np.uint32),
        ("det_offsets", np.uint32), ("det_meas", np.uint32), ("obs_offsets", np.uint32),
        ("obs_meas", np.uint32)))
    # numpy returns a NULL-free pointer only for non-empty arrays; pad empties.
    arrs = tuple(a if a.size else np.zeros(1, a.dtype) for a in arrs)
    types = (_u32p, _u8p, _u32p, _u32p, _i32p, _f64p, _u32p, _u8p, _f64p, _u32p, _u32p, _u32p, _u32p, _u32p,
             _u32p)
    v = CircuitView(c.num_qubits, c.num_layers, c.num_measurements, c.num_detectors, c.num_observables,
                    *(ptr(a, t) for a, t in zip(arrs, types)))
    return v, arrs


def copy_u64(p, n) -> np.ndarray:
    return np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, np.uint64)


def copy_u32(p, n) -> np.ndarray:
    return np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, np.uint32)


def copy_f64(p, n) -> np.ndarray:
    return np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, np.float64)

"""ctypes bindings of the two CPU checkers (TEST INFRASTRUCTURE).

* RefLib  -- the UNMODIFIED reference `demc` compiled from its own sources
  (oracle/Makefile -> oracle/_ref/libdemc_ref.so, glue in ref_capi.cpp).
* Port    -- the plain-C restatement oracle/demc_oracle.c
  (-> oracle/_build/libdemc_oracle.so).
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libdemc_ref.so"
PORT_SO = HERE / "_build" / "libdemc_oracle.so"


def build(ref: bool = True) -> None:
    have_ref = ref and Path("/root/reference/proj/core/src").exists()
    targets = ["port"] + (["ref"] if have_ref else [])
    # the reference's acceptance gate linked against the drop-in (needs libgreenpeas.so)
    if have_ref and (HERE.parent / "paper_2604_16613_b200" / "_lib" / "libgreenpeas.so").exists():
        targets.append("dropin")
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


class RefLib:
    def __init__(self):
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref)")
        L = C.CDLL(str(REF_SO))
        vp, sz = C.c_void_p, C.POINTER(C.c_size_t)
        L.ref_last_error.restype = C.c_char_p
        L.ref_free.argtypes = [vp]
        L.ref_circuit_parse.argtypes = [C.c_char_p]
        L.ref_circuit_parse.restype = vp
        L.ref_circuit_free.argtypes = [vp]
        L.ref_circuit_text.argtypes = [vp, sz]
        L.ref_circuit_text.restype = vp
        L.ref_compile.argtypes = [vp, C.c_int, C.c_uint32, C.POINTER(C.c_uint64), sz]
        L.ref_compile.restype = vp
        L.ref_oracle.argtypes = [vp, C.c_int, sz]
        L.ref_oracle.restype = vp
        L.ref_gen_surface.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_int]
        L.ref_gen_surface.restype = vp
        L.ref_gen_repetition.argtypes = [C.c_uint32, C.c_uint32, C.c_double]
        L.ref_gen_repetition.restype = vp
        L.ref_adaptive_shot.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, C.c_uint64, C.c_uint64,
                                        C.POINTER(vp), sz]
        L.ref_adaptive_shot.restype = vp
        L.ref_time_compile.argtypes = [vp, C.c_int, C.c_uint32, C.POINTER(C.c_uint64)]
        L.ref_time_compile.restype = C.c_int64
        L.ref_time_serialize.argtypes = [vp, C.c_int, C.c_uint32, C.POINTER(C.c_uint64)]
        L.ref_time_serialize.restype = C.c_int64
        L.ref_compile_pool.argtypes = [C.POINTER(vp), C.c_uint32, C.c_int, C.c_uint32, C.POINTER(C.c_uint64)]
        L.ref_compile_pool.restype = C.c_int64
        L.ref_gen_bb72_branches.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_double, C.c_double,
                                            C.c_uint64, C.c_uint32, C.POINTER(vp)]
        L.ref_gen_bb72_branches.restype = C.c_int
        L.ref_compile_digests.argtypes = [C.POINTER(vp), C.c_uint32, C.c_int, C.c_uint32, C.POINTER(C.c_uint64),
                                          C.POINTER(C.c_uint64)]
        L.ref_compile_digests.restype = C.c_int
        L.ref_dem_text_digest.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32]
        L.ref_dem_text_digest.restype = C.c_uint64
        L.ref_sample_fired.argtypes = [vp, C.c_uint64, C.c_uint32]
        L.ref_sample_fired.restype = C.c_int64
        self.L = L

    def _str(self, p, n) -> str:
        if not p:
            raise ValueError(self.L.ref_last_error().decode())
        s = C.string_at(p, n.value).decode()
        self.L.ref_free(p)
        return s

    def parse(self, text: str) -> "RefCircuit":
        h = self.L.ref_circuit_parse(text.encode())
        if not h:
            raise ValueError(self.L.ref_last_error().decode())
        return RefCircuit(self, h)

    def gen_surface(self, d, rounds, p, only_z=False) -> "RefCircuit":
        return RefCircuit(self, self.L.ref_gen_surface(d, rounds, p, int(only_z)))

    def gen_repetition(self, d, rounds, p) -> "RefCircuit":
        return RefCircuit(self, self.L.ref_gen_repetition(d, rounds, p))

    def adaptive_shot(self, d, rounds, refresh, p, seed, shot):
        txt = C.c_void_p()
        n = C.c_size_t()
        h = self.L.ref_adaptive_shot(d, rounds, refresh, p, seed, shot, C.byref(txt), C.byref(n))
        if not h:
            raise ValueError(self.L.ref_last_error().decode())
        return RefCircuit(self, h), self._str(txt.value, n)

    def gen_bb72_branches(self, first: int, count: int, rounds: int = 6, p: float = 1e-3,
                          check_prob: float = 0.5, seed: int = 1, threads: int = 0) -> list["RefCircuit"]:
        """Branch circuits b = first .. first + count - 1 as
        reference circuits: the repo's generator source compiled into this
        library, handed over as text to the reference's parse_circuit."""
        import os
        arr = (C.c_void_p * max(count, 1))()
        rc = self.L.ref_gen_bb72_branches(first, count, rounds, p, check_prob, seed, threads or os.cpu_count() or 1,
                                          arr)
        if rc:
            raise ValueError("branch generation failed")
        return [RefCircuit(self, arr[i]) for i in range(count)]

    def compile_digests(self, circuits, level: int, threads: int = 0):
        """Per circuit (hyperedges, DEM digest) of the reference compile_circuit."""
        import os
        n = len(circuits)
        arr = (C.c_void_p * max(n, 1))(*[c.h for c in circuits])
        e = np.zeros(max(n, 1), np.uint64)
        d = np.zeros(max(n, 1), np.uint64)
        rc = self.L.ref_compile_digests(arr, n, level, threads or os.cpu_count() or 1,
                                        e.ctypes.data_as(C.POINTER(C.c_uint64)),
                                        d.ctypes.data_as(C.POINTER(C.c_uint64)))
        if rc:
            raise ValueError("reference compile failed")
        return e[:n], d[:n]

    def dem_text_digest(self, text: str, num_detectors: int, num_observables: int) -> int:
        return int(self.L.ref_dem_text_digest(text.encode(), num_detectors, num_observables))

    def compile_pool(self, circuits, level: int, threads: int):
        arr = (C.c_void_p * len(circuits))(*[c.h for c in circuits])
        ns = C.c_uint64()
        e = self.L.ref_compile_pool(arr, len(circuits), level, threads, C.byref(ns))
        if e < 0:
            raise ValueError("reference compile failed")
        return int(e), int(ns.value)


class RefCircuit:
    def __init__(self, lib: RefLib, h):
        if not h:
            raise ValueError(lib.L.ref_last_error().decode())
        self.lib, self.h = lib, h

    def __del__(self):
        try:
            self.lib.L.ref_circuit_free(self.h)
        except Exception:
            pass

    def text(self) -> str:
        n = C.c_size_t()
        return self.lib._str(self.lib.L.ref_circuit_text(self.h, C.byref(n)), n)

    def compile(self, level: int, threads: int = 1):
        st = (C.c_uint64 * 5)()
        n = C.c_size_t()
        txt = self.lib._str(self.lib.L.ref_compile(self.h, level, threads, st, C.byref(n)), n)
        return txt, {"lower_ns": st[0], "traverse_ns": st[1], "reduce_ns": st[2], "total_ns": st[3],
                     "edges": st[4]}

    def oracle(self, level: int) -> str:
        n = C.c_size_t()
        return self.lib._str(self.lib.L.ref_oracle(self.h, level, C.byref(n)), n)

    def time_serialize(self, level: int, iters: int):
        """serialize_dem of this circuit's DEM, `iters` timed calls: (text length, ns)."""
        ns = (C.c_uint64 * iters)()
        n = self.lib.L.ref_time_serialize(self.h, level, iters, ns)
        if n < 0:
            raise ValueError(self.lib.L.ref_last_error().decode())
        return int(n), np.array(ns[:], dtype=np.uint64)

    def time_compile(self, level: int, iters: int):
        ns = (C.c_uint64 * iters)()
        e = self.lib.L.ref_time_compile(self.h, level, iters, ns)
        if e < 0:
            raise ValueError(self.lib.L.ref_last_error().decode())
        return int(e), np.array(ns[:], dtype=np.uint64)

    def sample_fired(self, seed: int, shots: int) -> int:
        return int(self.lib.L.ref_sample_fired(self.h, seed, shots))


class _OCircuit(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("num_qubits", "num_layers", "num_measurements", "num_detectors",
                                          "num_observables")] + [
        ("gate_offsets", C.POINTER(C.c_uint32)), ("gate_kind", C.POINTER(C.c_uint8)),
        ("gate_q0", C.POINTER(C.c_uint32)), ("gate_q1", C.POINTER(C.c_uint32)),
        ("gate_meas", C.POINTER(C.c_int32)), ("gate_flip", C.POINTER(C.c_double)),
        ("noise_offsets", C.POINTER(C.c_uint32)), ("noise_kind", C.POINTER(C.c_uint8)),
        ("noise_prob", C.POINTER(C.c_double)), ("noise_q0", C.POINTER(C.c_uint32)),
        ("noise_q1", C.POINTER(C.c_uint32)), ("det_offsets", C.POINTER(C.c_uint32)),
        ("det_meas", C.POINTER(C.c_uint32)), ("obs_offsets", C.POINTER(C.c_uint32)),
        ("obs_meas", C.POINTER(C.c_uint32))]


class _ODem(C.Structure):
    _fields_ = [("num_detectors", C.c_uint32), ("num_observables", C.c_uint32), ("num_edges", C.c_uint64),
                ("det_offsets", C.POINTER(C.c_uint64)), ("det_ids", C.POINTER(C.c_uint32)),
                ("obs_offsets", C.POINTER(C.c_uint64)), ("obs_ids", C.POINTER(C.c_uint32)),
                ("probs", C.POINTER(C.c_double)), ("num_sources", C.c_uint64),
                ("mem_offsets", C.POINTER(C.c_uint64)), ("mem_ids", C.POINTER(C.c_uint32))]


class Port:
    """The C restatement. Returns hyperedge lists [(dets, obs, p)] (+ members)."""

    def __init__(self):
        if not PORT_SO.exists():
            build(ref=False)
        L = C.CDLL(str(PORT_SO))
        L.oracle_compile.argtypes = [C.POINTER(_OCircuit), C.c_int, C.POINTER(_ODem)]
        L.oracle_forward.argtypes = [C.POINTER(_OCircuit), C.c_int, C.POINTER(_ODem)]
        L.oracle_dem_free.argtypes = [C.POINTER(_ODem)]
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_fnv1_64.argtypes = [C.POINTER(C.c_uint64), C.c_size_t]
        L.oracle_fnv1_64.restype = C.c_uint64
        L.oracle_merge_prob.argtypes = [C.c_double, C.c_double]
        L.oracle_merge_prob.restype = C.c_double
        self.L = L

    def _run(self, fn, circuit, level):
        names = [n for n, _ in _OCircuit._fields_[5:]]
        dts = [np.uint32, np.uint8, np.uint32, np.uint32, np.int32, np.float64, np.uint32, np.uint8, np.float64,
               np.uint32, np.uint32, np.uint32, np.uint32, np.uint32, np.uint32]
        keep = []
        ptrs = []
        for n, dt, (_, ct) in zip(names, dts, _OCircuit._fields_[5:]):
            a = np.ascontiguousarray(getattr(circuit, n), dtype=dt)
            if a.size == 0:
                a = np.zeros(1, dt)
            keep.append(a)
            ptrs.append(a.ctypes.data_as(ct))
        oc = _OCircuit(circuit.num_qubits, circuit.num_layers, circuit.num_measurements,
                       circuit.num_detectors, circuit.num_observables, *ptrs)
        od = _ODem()
        rc = fn(C.byref(oc), level, C.byref(od))
        if rc:
            raise ValueError(self.L.oracle_last_error().decode())
        E = od.num_edges
        edges, members = [], []
        for e in range(E):
            d = tuple(od.det_ids[k] for k in range(od.det_offsets[e], od.det_offsets[e + 1]))
            o = tuple(od.obs_ids[k] for k in range(od.obs_offsets[e], od.obs_offsets[e + 1]))
            edges.append((d, o, od.probs[e]))
            members.append([od.mem_ids[k] for k in range(od.mem_offsets[e], od.mem_offsets[e + 1])])
        S = od.num_sources
        self.L.oracle_dem_free(C.byref(od))
        return edges, members, S

    def compile(self, circuit, level):
        return self._run(self.L.oracle_compile, circuit, level)

    def forward(self, circuit, level):
        return self._run(self.L.oracle_forward, circuit, level)

    def fnv1_64(self, words) -> int:
        a = np.ascontiguousarray(words, dtype=np.uint64)
        if a.size == 0:
            return int(self.L.oracle_fnv1_64(None, 0))
        return int(self.L.oracle_fnv1_64(a.ctypes.data_as(C.POINTER(C.c_uint64)), a.size))

    def merge_prob(self, a, b) -> float:
        return float(self.L.oracle_merge_prob(a, b))


def parse_dem_text(text: str):
    """parse_dem (dem.cpp:158-197) to [(dets, obs, p)]; floats parse exactly."""
    out = []
    for line in text.splitlines():
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        toks = line.split()
        assert toks[0].startswith("error(") and toks[0].endswith(")"), line
        p = float(toks[0][6:-1])
        d = tuple(int(t[1:]) for t in toks[1:] if t[0] == "D")
        o = tuple(int(t[1:]) for t in toks[1:] if t[0] == "L")
        out.append((d, o, p))
    return out

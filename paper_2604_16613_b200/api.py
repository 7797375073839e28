"""Python mirror of the reference compile API over the C ABI.

    compile_circuit(circuit, level, threads=1, stats=None) -> Dem
        == demc::compile_circuit (/root/reference/proj/core/src/compile.cpp:23-53)

Same argument meaning and error behaviour: ValueError (the reference's
std::invalid_argument) with the reference's message text. The work runs on
the GPU through libgreenpeas.so; nothing here computes a DEM on the CPU.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from . import _native as N
from .circuit import Circuit


class CorrelationLevel(IntEnum):  # stepg.hpp:28
    L0 = 0
    L1 = 1
    L2 = 2


GP_OK, GP_ERR_INVALID_ARGUMENT, GP_ERR_CUDA, GP_ERR_OOM, GP_ERR_NO_DEVICE, GP_ERR_UNSUPPORTED = range(6)
OPT_FORCE_HASH_COLLISIONS, OPT_RECORD_SLOTS = 1, 2
GP_MEM_HOST, GP_MEM_DEVICE = 0, 1
NOISE_MODEL_PAPER, NOISE_MODEL_SI1000, NOISE_MODEL_UNIFORM = 0, 1, 2


class GreenpeasError(RuntimeError):
    pass


@dataclass
class Dem:
    """Flat demc::Dem (dem.hpp:38-52): hyperedges in canonical order."""

    num_detectors: int
    num_observables: int
    det_offsets: np.ndarray
    det_ids: np.ndarray
    obs_offsets: np.ndarray
    obs_ids: np.ndarray
    probs: np.ndarray

    @property
    def num_edges(self) -> int:
        return len(self.probs)

    def hyperedges(self):
        d, o = self.det_offsets, self.obs_offsets
        return [(tuple(int(x) for x in self.det_ids[d[e]:d[e + 1]]),
                 tuple(int(x) for x in self.obs_ids[o[e]:o[e + 1]]), float(self.probs[e]))
                for e in range(self.num_edges)]

    def view(self):
        arrs = (np.ascontiguousarray(self.det_offsets, np.uint32), np.ascontiguousarray(self.det_ids, np.uint32),
                np.ascontiguousarray(self.obs_offsets, np.uint32), np.ascontiguousarray(self.obs_ids, np.uint32),
                np.ascontiguousarray(self.probs, np.float64))
        arrs = tuple(a if a.size else np.zeros(1, a.dtype) for a in arrs)
        v = N.DemView(self.num_detectors, self.num_observables, self.num_edges,
                      N.ptr(arrs[0], N._u32p), N.ptr(arrs[1], N._u32p), N.ptr(arrs[2], N._u32p),
                      N.ptr(arrs[3], N._u32p), N.ptr(arrs[4], N._f64p))
        return v, arrs

    def digest(self) -> int:
        """gp_dem_digest: 64-bit hash of ids and probability bits (equal <=> same text)."""
        v, keep = self.view()
        return int(N.lib().gp_dem_digest(C.byref(v)))

    def to_text(self) -> str:
        """serialize_dem (dem.cpp:144-157), formatted natively with std::to_chars."""
        v, keep = self.view()
        n = C.c_size_t()
        p = N.lib().gp_serialize_dem(C.byref(v), C.byref(n))
        return N.take_string(p, n.value)


@dataclass
class PartialTable:
    """One fault-range shard's partial table (gp_partial_view):
    every nonempty source signature of the shard with its own probability,
    unfolded. Records: (64-bit id word, bits) pairs, detector d = bit d,
    observable o = bit D + o."""

    num_detectors: int
    num_observables: int
    probs: np.ndarray        # f64 [n]
    rec_offsets: np.ndarray  # u32 [n + 1]
    rec_words: np.ndarray    # u32 [r]
    rec_bits: np.ndarray     # u64 [r]

    @property
    def num_sources(self) -> int:
        return len(self.probs)

    def view(self):
        arrs = (np.ascontiguousarray(self.probs, np.float64), np.ascontiguousarray(self.rec_offsets, np.uint32),
                np.ascontiguousarray(self.rec_words, np.uint32), np.ascontiguousarray(self.rec_bits, np.uint64))
        arrs = tuple(a if a.size else np.zeros(1, a.dtype) for a in arrs)
        v = N.PartialView(self.num_detectors, self.num_observables, len(self.probs), len(self.rec_words),
                          GP_MEM_HOST, 0, N.ptr(arrs[0], N._f64p), N.ptr(arrs[1], N._u32p),
                          N.ptr(arrs[2], N._u32p), N.ptr(arrs[3], N._u64p))
        return v, arrs


class _CudaArray:
    """A raw device range as __cuda_array_interface__ (torch.as_tensor wraps it
    without a copy). Unsigned ids travel as same-width signed integers."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (int(ptr or 0), False),
                                         "version": 3, "strides": None}


@dataclass
class DevicePartialTable:
    """A partial table in device memory (GP_MEM_DEVICE) as torch tensors:
    probs f64, rec_offsets / rec_words int32 (u32 bits), rec_bits int64 (u64
    bits). Tensors returned by compile_shard(on_device=True) are views of the
    compiler's workspace: valid until its next call (clone to keep)."""

    num_detectors: int
    num_observables: int
    probs: object
    rec_offsets: object
    rec_words: object
    rec_bits: object

    @property
    def num_sources(self) -> int:
        return int(self.probs.numel())

    def arrays(self) -> dict:
        return {"probs": self.probs, "rec_offsets": self.rec_offsets, "rec_words": self.rec_words,
                "rec_bits": self.rec_bits}

    def view(self):
        ts = tuple(t.contiguous() for t in (self.probs, self.rec_offsets, self.rec_words, self.rec_bits))
        v = N.PartialView(self.num_detectors, self.num_observables, ts[0].numel(), ts[2].numel(), GP_MEM_DEVICE, 0,
                          C.cast(C.c_void_p(ts[0].data_ptr()), N._f64p), C.cast(C.c_void_p(ts[1].data_ptr()), N._u32p),
                          C.cast(C.c_void_p(ts[2].data_ptr()), N._u32p), C.cast(C.c_void_p(ts[3].data_ptr()), N._u64p))
        return v, ts


def _dem_slice(v, doff: np.ndarray, ooff: np.ndarray, lo: int, hi: int, nd: int, no: int) -> Dem:
    """Edges [lo, hi) of a flat DEM view (offset arrays already copied)."""
    E = hi - lo
    d0, d1, o0, o1 = int(doff[lo]), int(doff[hi]), int(ooff[lo]), int(ooff[hi])
    dids = np.ctypeslib.as_array(v.det_ids, shape=(d1,))[d0:d1].copy() if d1 > d0 else np.zeros(0, np.uint32)
    oids = np.ctypeslib.as_array(v.obs_ids, shape=(o1,))[o0:o1].copy() if o1 > o0 else np.zeros(0, np.uint32)
    probs = np.ctypeslib.as_array(v.probs, shape=(hi,))[lo:hi].copy() if E else np.zeros(0, np.float64)
    return Dem(nd, no, doff[lo:hi + 1] - np.uint32(d0), dids, ooff[lo:hi + 1] - np.uint32(o0), oids, probs)


def _dem_from_view(v, lo: int, hi: int, nd: int, no: int) -> Dem:
    doff = N.copy_u32(v.det_offsets, v.num_edges + 1) if v.num_edges else np.zeros(1, np.uint32)
    ooff = N.copy_u32(v.obs_offsets, v.num_edges + 1) if v.num_edges else np.zeros(1, np.uint32)
    return _dem_slice(v, doff, ooff, lo, hi, nd, no)


class Compiler:
    """One GPU context (stream, pinned arenas, device workspace). Not
    thread-safe: use one per host thread (compile_circuit does that)."""

    def __init__(self, device: int = 0):
        self._lib = N.lib()
        self._ctx = C.c_void_p()
        self.device = int(device)
        st = self._lib.gp_ctx_create(int(device), C.byref(self._ctx))
        if st != GP_OK:
            raise GreenpeasError(f"gp_ctx_create(device={device}) failed with status {st} "
                                 "(no CUDA device? there is no CPU fallback)")
        self.last_stats: dict = {}

    def close(self):
        if self._ctx:
            self._lib.gp_ctx_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, option: int, value: int) -> None:
        self._check(self._lib.gp_ctx_set_option(self._ctx, option, value))

    def _check(self, st: int) -> None:
        if st == GP_OK:
            return
        msg = self._lib.gp_last_error(self._ctx).decode()
        if st == GP_ERR_INVALID_ARGUMENT:
            raise ValueError(msg)
        raise GreenpeasError(f"status {st}: {msg}")

    def compile(self, circuit, level=CorrelationLevel.L0) -> Dem:
        v, keep = circuit.view() if hasattr(circuit, "view") else N.view_of(circuit)
        out = N.DemView()
        st = N.Stats()
        self._check(self._lib.gp_compile(self._ctx, C.byref(v), int(level), C.byref(out), C.byref(st)))
        self.last_stats = st.as_dict()
        return _dem_from_view(out, 0, int(out.num_edges), out.num_detectors, out.num_observables)

    def compile_shard(self, circuit, shard: int, nshards: int, level=CorrelationLevel.L0,
                      on_device: bool = False):
        """Fault-range shard `shard` of `nshards` (layers [l*k/n, l*(k+1)/n))
        of one circuit as a partial table (gp_compile_shard): a PartialTable
        in host memory, or with on_device a DevicePartialTable (torch views of
        the device workspace, ready for an NCCL gather)."""
        v, keep = circuit.view() if hasattr(circuit, "view") else N.view_of(circuit)
        out = N.PartialView()
        st = N.Stats()
        mem = GP_MEM_DEVICE if on_device else GP_MEM_HOST
        self._check(self._lib.gp_compile_shard(self._ctx, C.byref(v), int(level), int(shard), int(nshards), mem,
                                               C.byref(out), C.byref(st)))
        self.last_stats = st.as_dict()
        n, r = int(out.num_sources), int(out.num_records)
        if on_device:
            import torch
            dev = torch.device("cuda", self.device)

            def wrap(ptr, count, ts):
                if count == 0:
                    return torch.zeros(0, dtype={"<f8": torch.float64, "<i4": torch.int32,
                                                 "<i8": torch.int64}[ts], device=dev)
                return torch.as_tensor(_CudaArray(C.cast(ptr, C.c_void_p).value, count, ts), device=dev)
            return DevicePartialTable(int(out.num_detectors), int(out.num_observables), wrap(out.probs, n, "<f8"),
                                      wrap(out.rec_offsets, n + 1, "<i4"), wrap(out.rec_words, r, "<i4"),
                                      wrap(out.rec_bits, r, "<i8"))
        return PartialTable(
            int(out.num_detectors), int(out.num_observables), N.copy_f64(out.probs, n) if n else
            np.zeros(0, np.float64), N.copy_u32(out.rec_offsets, n + 1), N.copy_u32(out.rec_words, r) if r else
            np.zeros(0, np.uint32), N.copy_u64(out.rec_bits, r) if r else np.zeros(0, np.uint64))

    def merge_partials(self, parts: list) -> Dem:
        """The DEM of the union of partial tables (gp_merge_partials): equal to
        compile() of the whole circuit when the parts cover every shard."""
        arr = (N.PartialView * len(parts))()
        keep = []
        if any(isinstance(t, DevicePartialTable) for t in parts):
            import torch
            torch.cuda.synchronize(self.device)  # producers of device tables ran on torch's streams
        for i, t in enumerate(parts):
            v, k = t.view()
            arr[i] = v
            keep.append(k)
        out = N.DemView()
        st = N.Stats()
        self._check(self._lib.gp_merge_partials(self._ctx, arr, len(parts), C.byref(out), C.byref(st)))
        self.last_stats = st.as_dict()
        return _dem_from_view(out, 0, int(out.num_edges), out.num_detectors, out.num_observables)

    def replay(self, iterations: int = 1, flush_l2: bool = False) -> dict:
        """Re-runs the device pipeline on the last uploaded batch (inputs and
        outputs resident in HBM); returns summed device times in ns."""
        st = N.Stats()
        self._check(self._lib.gp_replay(self._ctx, iterations, int(flush_l2), C.byref(st)))
        return st.as_dict()

    def profile_stages(self) -> dict:
        ns = (C.c_uint64 * 32)()
        names = (C.c_char_p * 32)()
        n = self._lib.gp_profile_stages(self._ctx, ns, names, 32)
        return {names[i].decode(): int(ns[i]) for i in range(n)}

    def compile_batch_raw(self, views, level=CorrelationLevel.L0):
        """Batch compile of prepared CircuitView array; returns (DemBatchView, stats)."""
        out = N.DemBatchView()
        st = N.Stats()
        self._check(self._lib.gp_compile_batch(self._ctx, views, len(views), int(level), C.byref(out),
                                               C.byref(st)))
        self.last_stats = st.as_dict()
        return out, self.last_stats

    def compile_bb_branches_raw(self, spec: "N.BBSpec", first: int, count: int,
                                level=CorrelationLevel.L0):
        """Branch circuits generated on the device (gp_compile_bb_branches):
        seeds in, batch DEM out; returns (DemBatchView, stats)."""
        out = N.DemBatchView()
        st = N.Stats()
        self._check(self._lib.gp_compile_bb_branches(self._ctx, C.byref(spec), first, count, int(level),
                                                     C.byref(out), C.byref(st)))
        self.last_stats = st.as_dict()
        return out, self.last_stats

    @staticmethod
    def batch_digests(out) -> np.ndarray:
        """Per-circuit gp_dem_digest of a DemBatchView (host threads)."""
        d = np.zeros(max(int(out.num_circuits), 1), np.uint64)
        N.lib().gp_dem_batch_digest(C.byref(out), N.ptr(d, N._u64p))
        return d[:int(out.num_circuits)]

    def compile_batch(self, circuits, level=CorrelationLevel.L0) -> list[Dem]:
        keep = []
        arr = (N.CircuitView * len(circuits))()
        for i, c in enumerate(circuits):
            v, k = c.view() if hasattr(c, "view") else N.view_of(c)
            arr[i] = v
            keep.append(k)
        out, _ = self.compile_batch_raw(arr, level)
        eo = N.copy_u64(out.edge_offsets, len(circuits) + 1)
        E = int(out.num_edges)
        doff = N.copy_u32(out.det_offsets, E + 1) if E else np.zeros(1, np.uint32)
        ooff = N.copy_u32(out.obs_offsets, E + 1) if E else np.zeros(1, np.uint32)
        return [_dem_slice(out, doff, ooff, int(eo[i]), int(eo[i + 1]), int(out.num_detectors[i]),
                           int(out.num_observables[i])) for i in range(len(circuits))]


_tls = threading.local()


def _thread_compiler(device: int = 0) -> Compiler:
    c = getattr(_tls, "compiler", None)
    if c is None:
        c = _tls.compiler = Compiler(device)
    return c


def compile_circuit(circuit, level=CorrelationLevel.L0, threads: int = 1, stats: dict | None = None) -> Dem:
    """Drop-in for demc::compile_circuit (compile.hpp:35-36). `threads` is
    accepted for signature parity; the output never depends on it."""
    del threads
    comp = _thread_compiler()
    d = comp.compile(circuit, level)
    if stats is not None:
        stats.update(comp.last_stats)
    return d


class GenCircuit:
    """Owning native circuit produced by a gp_gen_* generator."""

    def __init__(self, handle):
        if not handle:
            raise ValueError("generator rejected its parameters")
        self._h = C.c_void_p(handle)
        v = N.lib().gp_circuit_get_view(self._h)
        self._view = v

    def view(self):
        return self._view, (self,)

    @property
    def num_qubits(self):
        return self._view.num_qubits

    @property
    def num_layers(self):
        return self._view.num_layers

    @property
    def num_measurements(self):
        return self._view.num_measurements

    @property
    def num_detectors(self):
        return self._view.num_detectors

    @property
    def num_observables(self):
        return self._view.num_observables

    def to_text(self) -> str:
        n = C.c_size_t()
        p = N.lib().gp_circuit_serialize(self._h, C.byref(n))
        return N.take_string(p, n.value)

    def to_circuit(self) -> Circuit:
        v = self._view
        L, D, O = v.num_layers, v.num_detectors, v.num_observables
        goff = N.copy_u32(v.gate_offsets, L + 1)
        noff = N.copy_u32(v.noise_offsets, L + 1)
        doff = N.copy_u32(v.det_offsets, D + 1)
        ooff = N.copy_u32(v.obs_offsets, O + 1)
        G, NN = int(goff[-1]), int(noff[-1])

        def arr(p, n, dt):
            return np.ctypeslib.as_array(p, shape=(n,)).astype(dt) if n else np.zeros(0, dt)

        return Circuit(v.num_qubits, v.num_measurements, goff, arr(v.gate_kind, G, np.uint8),
                       arr(v.gate_q0, G, np.uint32), arr(v.gate_q1, G, np.uint32), arr(v.gate_meas, G, np.int32),
                       arr(v.gate_flip, G, np.float64), noff, arr(v.noise_kind, NN, np.uint8),
                       arr(v.noise_prob, NN, np.float64), arr(v.noise_q0, NN, np.uint32),
                       arr(v.noise_q1, NN, np.uint32), doff, arr(v.det_meas, int(doff[-1]), np.uint32), ooff,
                       arr(v.obs_meas, int(ooff[-1]), np.uint32))

    def __del__(self):
        try:
            N.lib().gp_circuit_free(self._h)
        except Exception:
            pass


def circuit_metrics(circuit, level) -> dict:
    """SURVEY.md 8d inputs of the algorithmic-bytes formula for one circuit."""
    v, keep = circuit.view() if hasattr(circuit, "view") else N.view_of(circuit)
    m = N.Metrics()
    N.lib().gp_circuit_metrics(C.byref(v), int(level), C.byref(m))
    return {n: int(getattr(m, n)) for n, _ in m._fields_}


def algorithmic_bytes(metrics: dict, edges: int, ids: int) -> dict:
    """B_alg = 8N + 8W(N + M + N_e + C) + 8S + E(8 + 4 w), split
    into the traversal part (dense Alg. 1 + leaf init + signature gather) and
    the reduce part (probabilities in, compact DEM out); E*4*w = 4*ids."""
    N_, W, M = metrics["base_nodes"], metrics["words"], metrics["measurements"]
    trav = 8 * N_ + 8 * W * (N_ + M + metrics["succ_refs"] + metrics["source_rows"])
    red = 8 * metrics["sources"] + 8 * edges + 4 * ids
    return {"traverse": trav, "reduce": red, "total": trav + red}


class CircuitParseError(ValueError):
    """gp_parse_circuit's error: the reference's message ("line N: ..." or
    "layer L: ...")."""


def parse_circuit_native(text: str) -> "GenCircuit":
    """parse_circuit + validate_layers (circuit.cpp:107-326) in native code
    (gp_parse_circuit; parallel on the host pool for large texts)."""
    data = text.encode()
    err = C.c_void_p()
    h = N.lib().gp_parse_circuit(data, len(data), C.byref(err))
    if not h:
        msg = C.string_at(err.value).decode() if err.value else "parse failed"
        if err.value:
            N.lib().gp_free(err)
        raise CircuitParseError(msg)
    return GenCircuit(h)


def gen_repetition(d: int, rounds: int, p: float) -> GenCircuit:
    return GenCircuit(N.lib().gp_gen_repetition(d, rounds, p))


def gen_surface(d: int, rounds: int, p: float, noise_model: int = NOISE_MODEL_PAPER,
                only_z: bool = False) -> GenCircuit:
    return GenCircuit(N.lib().gp_gen_surface(d, rounds, p, noise_model, int(only_z)))


def gen_bb(l: int, m: int, a=(3, 1, 2), b=(3, 1, 2), rounds: int = 12, p: float = 1e-3,
           noise_model: int = NOISE_MODEL_UNIFORM, check_prob: float = 1.0, refresh: int = 0,
           seed: int = 1, branch: int = 0) -> GenCircuit:
    A = (C.c_uint32 * 3)(*a)
    B = (C.c_uint32 * 3)(*b)
    return GenCircuit(N.lib().gp_gen_bb(l, m, A, B, rounds, p, noise_model, check_prob, refresh, seed, branch))


def gen_bb144(rounds: int = 12, p: float = 1e-3, noise_model: int = NOISE_MODEL_UNIFORM) -> GenCircuit:
    """Gross code [[144,12,12]]: A = x^3 + y + y^2, B = y^3 + x + x^2, (l, m) = (12, 6)."""
    return gen_bb(12, 6, rounds=rounds, p=p, noise_model=noise_model)


def bb_spec(l: int, m: int, a=(3, 1, 2), b=(3, 1, 2), rounds: int = 12, p: float = 1e-3,
            noise_model: int = NOISE_MODEL_UNIFORM, check_prob: float = 1.0, refresh: int = 0,
            seed: int = 1) -> "N.BBSpec":
    """gp_bb_spec of gen_bb's circuits (for Compiler.compile_bb_branches_raw)."""
    return N.BBSpec(l, m, (C.c_uint32 * 3)(*a), (C.c_uint32 * 3)(*b), rounds, refresh, noise_model, 0, p,
                    check_prob, seed)


def bb72_branch_spec(rounds: int = 6, p: float = 1e-3, check_prob: float = 0.5, seed: int = 1) -> "N.BBSpec":
    """gp_bb_spec of gen_bb72_branch."""
    return bb_spec(6, 6, rounds=rounds, p=p, noise_model=NOISE_MODEL_PAPER, check_prob=check_prob,
                   refresh=max(1, rounds // 2), seed=seed)


def gen_bb72_branch(branch: int, rounds: int = 6, p: float = 1e-3, check_prob: float = 0.5,
                    seed: int = 1) -> GenCircuit:
    """[[72,12,6]] adaptive branch circuit: full rounds at
    r = 0, the last round and every refresh = d/2 round; otherwise each check
    runs with probability check_prob drawn from mt19937_64(seed_seq{seed, seed>>32,
    branch, branch>>32}). Paper noise model NoiseModel{p} (codes.hpp:30-39)."""
    return gen_bb(6, 6, rounds=rounds, p=p, noise_model=NOISE_MODEL_PAPER, check_prob=check_prob,
                  refresh=max(1, rounds // 2), seed=seed, branch=branch)

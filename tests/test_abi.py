"""CPU: the C-ABI library loads, exports every entry point include/greenpeas.h
declares (plus the demc::compile_circuit C++ shim), and its host-only
functions (DEM formatting, generators) behave. No device compute here."""

import ctypes as C
import re
import subprocess

import numpy as np
import pytest

import paper_2604_16613_b200 as gp
from paper_2604_16613_b200 import _native as N

from .conftest import ROOT


def declared_symbols():
    hdr = (ROOT / "include" / "greenpeas.h").read_text()
    return sorted(set(re.findall(r"\b(gp_[a-z0-9_]+)\s*\(", hdr)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("gp_ctx_create", "gp_ctx_destroy", "gp_compile", "gp_compile_batch", "gp_last_error",
              "gp_serialize_dem"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), f"{s} not exported by {N.LIB_PATH}"


def test_cpp_shim_symbol_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", "-C", str(N.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    assert "demc::compile_circuit(demc::Circuit const&, demc::CorrelationLevel, unsigned int, demc::CompileStats*)" in out
    assert "demc::serialize_dem[abi:cxx11](demc::Dem const&)" in out


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def dem_from_edges(edges, nd, no):
    doff, dids, ooff, oids, probs = [0], [], [0], [], []
    for d, o, p in edges:
        dids += d
        oids += o
        doff.append(len(dids))
        ooff.append(len(oids))
        probs.append(p)
    return gp.Dem(nd, no, np.array(doff, np.uint64), np.array(dids, np.uint32), np.array(ooff, np.uint64),
                  np.array(oids, np.uint32), np.array(probs, np.float64))


def test_serialize_known_answer():
    """test_dem.cpp:103-110."""
    d = dem_from_edges([((0, 1), (), 0.125), ((1,), (0,), 0.0625)], 2, 1)
    assert d.to_text() == "error(0.125) D0 D1\nerror(0.0625) D1 L0\n"


def test_serialize_is_byte_identical_on_fixtures():
    from oracle.bindings import parse_dem_text
    for fx in sorted((ROOT / "tests" / "golden" / "fixtures").iterdir()):
        text = (fx / "expected.dem").read_text()
        c = gp.parse_circuit((fx / "circuit.txt").read_text())
        d = dem_from_edges(parse_dem_text(text), c.num_detectors, c.num_observables)
        assert d.to_text() == text


def test_shortest_round_trip_formatting():
    d = dem_from_edges([((0,), (), 5.333084451081371e-05), ((1,), (), 1e-4), ((2,), (), 0.06593723337664)], 3, 0)
    assert d.to_text() == "error(5.333084451081371e-05) D0\nerror(1e-04) D1\nerror(0.06593723337664) D2\n"


def test_context_without_device_fails_loudly():
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("a GPU is present")
    ctx = C.c_void_p()
    assert N.lib().gp_ctx_create(0, C.byref(ctx)) == 4  # GP_ERR_NO_DEVICE
    with pytest.raises(gp.GreenpeasError):
        gp.Compiler(0)


def _dem_view(edges):
    doff = np.zeros(len(edges) + 1, np.uint32)
    ooff = np.zeros(len(edges) + 1, np.uint32)
    dids, oids = [], []
    pr = np.zeros(max(len(edges), 1))
    for i, (d, o, p) in enumerate(edges):
        dids += d
        oids += o
        doff[i + 1], ooff[i + 1], pr[i] = len(dids), len(oids), p
    arrs = (doff, np.array(dids + [0], np.uint32), ooff, np.array(oids + [0], np.uint32), pr)
    u32 = C.POINTER(C.c_uint32)
    v = N.DemView(0, 0, len(edges), *(a.ctypes.data_as(u32) for a in arrs[:4]),
                  arrs[4].ctypes.data_as(C.POINTER(C.c_double)))
    return v, arrs


def _serialize(v):
    n = C.c_size_t()
    return N.take_string(N.lib().gp_serialize_dem(C.byref(v), C.byref(n)), n.value)


def test_serialize_large_dem_byte_identical_to_reference():
    """gp_serialize_dem on a DEM large enough for the parallel pieces and the
    repeated-probability text cache (surface d11 SI1000 L2: 24k hyperedges,
    64 distinct probabilities) equals the reference's serialize_dem."""
    from oracle.bindings import RefLib, parse_dem_text
    g = gp.gen_surface(11, 11, 1e-3, gp.NOISE_MODEL_SI1000)
    text, _ = RefLib().parse(g.to_text()).compile(2)
    body = "".join(line + "\n" for line in text.splitlines() if line.startswith("error"))
    v, keep = _dem_view(parse_dem_text(text))
    assert _serialize(v) == body


def test_serialize_many_distinct_probabilities_round_trip():
    """Colliding and repeated probabilities in the text cache: every printed
    probability parses back to its own double, ids intact."""
    rng = np.random.default_rng(5)
    pool = np.concatenate([rng.random(300) * 1e-2, [0.0, -0.0, 1.0, 5e-324, 1e-300, 0.5]])
    edges = [((int(i), int(i) + 3), (1,) if i % 7 == 0 else (), float(pool[rng.integers(pool.size)]))
             for i in range(20000)]
    v, keep = _dem_view(edges)
    lines = _serialize(v).splitlines()
    assert len(lines) == len(edges)
    for line, (d, o, p) in zip(lines, edges):
        head, *ids = line.split(" ")
        q = float(head[6:-1])
        assert q == p and np.signbit(q) == np.signbit(p), (line, p)
        assert ids == [f"D{x}" for x in d] + [f"L{x}" for x in o]

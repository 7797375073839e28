"""GPU parity: the sm_100a path (through the C ABI) against the reference.

Checks, in order of strength:
* byte-identical serialize_dem text vs the reference's golden fixtures and
  vs reference outputs committed under tests/golden/generated;
* at BASELINE.json full sizes: sha256 of the serialized DEM == the sha256 of
  the reference's own output on the same circuit (tests/golden/full_size.json);
* vs the C restatement oracle on edge cases the reference tests exercise
  (collisions, zero probabilities, empty / noiseless circuits, errors).
Bit-exact comparison throughout: ids exact and fp64 probabilities equal.
"""

import hashlib
import json
import subprocess
import threading

import numpy as np
import pytest

import paper_2604_16613_b200 as gp
from oracle.bindings import parse_dem_text

from .conftest import FIXTURES, GOLDEN, ROOT, fixture_case

pytestmark = pytest.mark.gpu

FULL = json.loads((GOLDEN / "full_size.json").read_text())


def sha(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()


@pytest.mark.parametrize("fx", FIXTURES, ids=lambda p: p.name)
def test_fixture_byte_identical(compiler, fx):
    circuit, level, text, golden = fixture_case(fx)
    dem = compiler.compile(circuit, level)
    assert dem.hyperedges() == golden
    assert dem.to_text() == text


@pytest.mark.parametrize("name", ["rep_d3_r2", "rep_d5_r3", "surface_d3_r3", "surface_d4_r2",
                                  "surface_d5_r5_si1000", "surface_d5_r3_onlyz"])
@pytest.mark.parametrize("level", [0, 1, 2])
def test_generated_golden_byte_identical(compiler, name, level):
    d = GOLDEN / "generated"
    circuit = gp.parse_circuit((d / f"{name}.circuit.txt").read_text())
    assert compiler.compile(circuit, level).to_text() == (d / f"{name}.L{level}.dem").read_text()


FULL_MAKERS = {
    "bb72_r2_uniform": lambda: gp.gen_bb(6, 6, rounds=2, p=1e-3),
    "bb72_branch3_r4": lambda: gp.gen_bb72_branch(3, rounds=4),
    "surface_d3_r3_paper": lambda: gp.gen_surface(3, 3, 1e-3),
    "surface_d11_r11_si1000": lambda: gp.gen_surface(11, 11, 1e-3, gp.NOISE_MODEL_SI1000),
    "bb144_r12_uniform": lambda: gp.gen_bb144(12, 1e-3),
    "surface_d25_r25_paper": lambda: gp.gen_surface(25, 25, 1e-3),
}
FULL_CASES = [(n, int(lv)) for n in FULL_MAKERS for lv in FULL[n]["levels"]]


@pytest.mark.parametrize("name,level", FULL_CASES, ids=[f"{n}-L{lv}" for n, lv in FULL_CASES])
def test_full_size_matches_reference_hash(compiler, name, level):
    g = FULL_MAKERS[name]()
    assert sha(g.to_text()) == FULL[name]["circuit_sha256"], "generator drifted from the golden circuit"
    dem = compiler.compile(g, level)
    want = FULL[name]["levels"][str(level)]
    assert dem.num_edges == want["edges"]
    assert sha(dem.to_text()) == want["dem_sha256"]


def test_branch_batch_matches_reference_hashes(compiler):
    info = FULL["bb72_branches_r6_L0"]["branches"]
    gens = [gp.gen_bb72_branch(b["branch"]) for b in info]
    for g, b in zip(gens, info):
        assert sha(g.to_text()) == b["circuit_sha256"]
    dems = compiler.compile_batch(gens, 0)
    for d, b in zip(dems, info):
        assert d.num_edges == b["edges"]
        assert sha(d.to_text()) == b["dem_sha256"]


def test_batch_equals_single_compiles(compiler, port):
    gens = [gp.gen_surface(3, 2, 1e-3), gp.gen_repetition(3, 2, 1e-3), gp.parse_circuit("H 0\nTICK\nM 0\n"),
            gp.gen_bb(6, 6, rounds=1, p=2e-3), gp.parse_circuit("R 0\nX_ERROR(0.1) 0\nTICK\nM 0\nDETECTOR rec[-1]\n"),
            gp.gen_surface(5, 2, 1e-3, gp.NOISE_MODEL_SI1000)]
    for level in (0, 1, 2):
        batch = compiler.compile_batch(gens, level)
        for g, d in zip(gens, batch):
            c = g.to_circuit() if hasattr(g, "to_circuit") else g
            assert d.hyperedges() == port.compile(c, level)[0]
            assert d.hyperedges() == compiler.compile(g, level).hyperedges()


@pytest.mark.parametrize("level", [0, 1, 2])
def test_small_generated_vs_oracle(compiler, port, level):
    for g in (gp.gen_surface(7, 3, 1e-3), gp.gen_bb72_branch(21, rounds=4), gp.gen_repetition(9, 5, 3e-3),
              gp.gen_surface(4, 4, 2e-3, gp.NOISE_MODEL_UNIFORM)):
        assert compiler.compile(g, level).hyperedges() == port.compile(g.to_circuit(), level)[0]


def test_forced_hash_collisions_never_merge(port):
    """test_dem.cpp:94-101 via the context's collision hook: every signature
    hashes to one key; grouping must still follow full comparison."""
    comp = gp.Compiler(0)
    comp.set_option(gp.OPT_FORCE_HASH_COLLISIONS, 1)
    for g in (gp.gen_surface(3, 3, 1e-3), gp.gen_repetition(5, 2, 1e-3)):
        for level in (0, 2):
            assert comp.compile(g, level).hyperedges() == port.compile(g.to_circuit(), level)[0]


def test_record_slot_overflow_recovers(port):
    """One inline slot per source: multi-word signatures overflow, the
    context grows its slots and re-runs; output unchanged."""
    comp = gp.Compiler(0)
    comp.set_option(gp.OPT_RECORD_SLOTS, 1)
    g = gp.gen_surface(11, 3, 1e-3)
    assert comp.compile(g, 2).hyperedges() == port.compile(g.to_circuit(), 2)[0]


def test_zero_probability_sources_retained(compiler, port):
    """test_stepg.cpp:78-83: X_ERROR(0) is a source; its edge has p = 0."""
    c = gp.parse_circuit("R 0\nX_ERROR(0) 0\nTICK\nM 0\nDETECTOR rec[-1]\n")
    got = compiler.compile(c, 0).hyperedges()
    assert got == port.compile(c, 0)[0] == [((0,), (), 0.0)]


def test_noiseless_and_empty_circuits(compiler):
    assert compiler.compile(gp.gen_surface(3, 2, 0.0), 2).num_edges == 0
    assert compiler.compile(gp.parse_circuit("H 0\n"), 0).num_edges == 0
    assert compiler.compile(gp.parse_circuit("X_ERROR(0.1) 0\nTICK\nM 0\n"), 0).num_edges == 0


def test_observable_only_edges_and_same_qubit_pairs(compiler, port):
    text = ("R 0 1\nTICK\nDEPOLARIZE2(0.3) 0 0\nX_ERROR(0.2) 1\nTICK\nM(0.05) 0 1\n"
            "OBSERVABLE_INCLUDE(0) rec[-1]\nOBSERVABLE_INCLUDE(1)\n")
    c = gp.parse_circuit(text)
    for level in (0, 1, 2):
        assert compiler.compile(c, level).hyperedges() == port.compile(c, level)[0]


def test_invalid_argument_messages(compiler):
    """eec.cpp:44-46 / 52-54 and stepg.cpp:172-174, verbatim."""
    c = gp.parse_circuit("M 0\nDETECTOR rec[-1]\nOBSERVABLE_INCLUDE(0) rec[-1]\n")
    bad = gp.Circuit(**{**c.__dict__, "det_meas": np.array([7], np.uint32)})
    with pytest.raises(ValueError, match="^detector references a measurement without a leaf$"):
        compiler.compile(bad, 0)
    bad = gp.Circuit(**{**c.__dict__, "obs_meas": np.array([7], np.uint32)})
    with pytest.raises(ValueError, match="^observable references a measurement without a leaf$"):
        compiler.compile(bad, 0)
    huge = gp.Circuit(**{**c.__dict__, "num_qubits": 1 << 27,
                         "gate_offsets": np.zeros(6, np.uint32), "noise_offsets": np.zeros(6, np.uint32),
                         "gate_kind": np.zeros(0, np.uint8), "gate_q0": np.zeros(0, np.uint32),
                         "gate_q1": np.zeros(0, np.uint32), "gate_meas": np.zeros(0, np.int32),
                         "gate_flip": np.zeros(0), "num_measurements": 0,
                         "det_offsets": np.zeros(1, np.uint32), "det_meas": np.zeros(0, np.uint32),
                         "obs_offsets": np.zeros(1, np.uint32), "obs_meas": np.zeros(0, np.uint32)})
    with pytest.raises(ValueError, match="^circuit exceeds 32-bit node index space$"):
        compiler.compile(huge, 2)
    # the context stays usable after an error
    assert compiler.compile(gp.gen_surface(3, 2, 1e-3), 0).num_edges == 46


def test_repeatable_and_schedule_independent(compiler):
    """acceptance.cpp:182-201: 20 repeats byte-identical; `threads` is inert."""
    g = gp.gen_surface(5, 2, 1e-3)
    first = compiler.compile(g, 2).to_text()
    for _ in range(20):
        assert compiler.compile(g, 2).to_text() == first
    assert gp.compile_circuit(g, 2, threads=32).to_text() == first


def test_concurrent_host_threads(port):
    """Reentrancy: one context per host thread."""
    g = gp.gen_surface(5, 3, 1e-3)
    want = port.compile(g.to_circuit(), 1)[0]
    errs = []

    def work():
        try:
            for _ in range(5):
                assert gp.compile_circuit(g, 1).hyperedges() == want
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=work) for _ in range(4)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert not errs


def test_stats_are_filled(compiler):
    stats = {}
    gp.compile_circuit(gp.gen_surface(5, 5, 1e-3), 2, stats=stats)
    assert stats["total_ns"] > 0 and stats["kernel_ns"] > 0 and stats["num_sources"] > 0
    assert stats["total_ns"] >= stats["kernel_ns"]


CPP_MAIN = r"""
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <stdexcept>
#include "demc/compile.hpp"
// Reads the flat dump written by the test and compiles it through the
// drop-in demc::compile_circuit (libgreenpeas), printing serialize_dem.
int main(int argc, char **argv) {
    std::ifstream in(argv[1]);
    int level = std::atoi(argv[2]);
    demc::Circuit c;
    std::string tag;
    c.layers.emplace_back();
    while (in >> tag) {
        if (tag == "Q") in >> c.num_qubits >> c.num_measurements;
        else if (tag == "L") c.layers.emplace_back();
        else if (tag == "G") {
            int k; demc::GateOp g{}; in >> k >> g.q0 >> g.q1 >> g.meas_index >> g.flip_prob;
            g.kind = (demc::GateKind)k; c.layers.back().gates.push_back(g);
        } else if (tag == "N") {
            int k; demc::NoiseOp n{}; in >> k >> n.prob >> n.q0 >> n.q1;
            n.kind = (demc::NoiseKind)k; c.layers.back().noise.push_back(n);
        } else if (tag == "D" || tag == "O") {
            size_t cnt; in >> cnt; std::vector<uint32_t> ms(cnt);
            for (auto &m : ms) in >> m;
            if (tag == "D") c.detectors.push_back({(uint32_t)c.detectors.size(), ms});
            else c.observables.push_back({(uint32_t)c.observables.size(), ms});
        }
    }
    c.layers.pop_back();
    try {
        demc::CompileStats st;
        demc::Dem d = demc::compile_circuit(c, (demc::CorrelationLevel)level, 1, &st);
        std::cout << demc::serialize_dem(d);
        std::cerr << "total_ns=" << st.total_ns << "\n";
    } catch (const std::invalid_argument &e) {
        std::cout << "invalid_argument: " << e.what() << "\n";
    }
    return 0;
}
"""


def dump_flat(c, path):
    lines = [f"Q {c.num_qubits} {c.num_measurements}"]
    for i in range(c.num_layers):
        for g in range(c.gate_offsets[i], c.gate_offsets[i + 1]):
            lines.append(f"G {c.gate_kind[g]} {c.gate_q0[g]} {c.gate_q1[g]} {c.gate_meas[g]} {float(c.gate_flip[g])!r}")
        for o in range(c.noise_offsets[i], c.noise_offsets[i + 1]):
            lines.append(f"N {c.noise_kind[o]} {float(c.noise_prob[o])!r} {c.noise_q0[o]} {c.noise_q1[o]}")
        lines.append("L")
    for ms in c.detectors():
        lines.append("D " + " ".join(map(str, [len(ms), *ms])))
    for ms in c.observables():
        lines.append("O " + " ".join(map(str, [len(ms), *ms])))
    path.write_text("\n".join(lines) + "\n")


def test_cpp_dropin_shim(tmp_path):
    """A C++ caller of the reference API links libgreenpeas unchanged."""
    from paper_2604_16613_b200._native import LIB_PATH
    src = tmp_path / "main.cpp"
    src.write_text(CPP_MAIN)
    exe = tmp_path / "dropin"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(src), str(LIB_PATH),
                    f"-Wl,-rpath,{LIB_PATH.parent}", "-o", str(exe)], check=True)
    for fx in FIXTURES:
        circuit, level, text, _ = fixture_case(fx)
        dump_flat(circuit, tmp_path / "c.txt")
        out = subprocess.run([str(exe), str(tmp_path / "c.txt"), str(level)], capture_output=True, text=True,
                             check=True)
        assert out.stdout == text, fx.name
    circuit, _, _, _ = fixture_case(FIXTURES[0])
    bad = gp.Circuit(**{**circuit.__dict__, "det_meas": circuit.det_meas + 1000})
    dump_flat(bad, tmp_path / "bad.txt")
    out = subprocess.run([str(exe), str(tmp_path / "bad.txt"), "0"], capture_output=True, text=True, check=True)
    assert out.stdout == "invalid_argument: detector references a measurement without a leaf\n"


def test_many_distinct_probabilities_use_wide_mode(compiler, port):
    """Distinct noise probabilities: up to 16383 per batch go through the
    packer's dictionary (14-bit table index); beyond that the batch is packed
    again with per-op fp64 probabilities. Results unchanged either way."""
    import random
    rng = random.Random(5)
    g = gp.gen_surface(5, 3, 1e-3).to_circuit()
    g.noise_prob = np.array([rng.uniform(1e-4, 3e-3) for _ in g.noise_prob])
    for level in (0, 2):
        assert compiler.compile(g, level).hyperedges() == port.compile(g, level)[0]
    small = gp.gen_surface(3, 2, 1e-3).to_circuit()
    batch = compiler.compile_batch([g, small], 1)
    assert batch[0].hyperedges() == port.compile(g, 1)[0]
    assert batch[1].hyperedges() == port.compile(small, 1)[0]
    # two circuits of ~14k distinct values each: the batch overflows the table
    big = []
    for seed in (1, 2):
        c = gp.gen_surface(11, 11, 1e-3).to_circuit()
        r = random.Random(seed)
        c.noise_prob = np.array([r.uniform(1e-4, 3e-3) for _ in c.noise_prob])
        big.append(c)
    assert len(set(big[0].noise_prob.tolist()) | set(big[1].noise_prob.tolist())) > 16383
    dems = compiler.compile_batch(big, 0)
    assert compiler.last_stats["h2d_bytes"] > 8 * (len(big[0].noise_prob) + len(big[1].noise_prob))  # fp64 per op
    for c, d in zip(big, dems):
        assert d.hyperedges() == port.compile(c, 0)[0]
        assert d.to_text() == compiler.compile(c, 0).to_text()  # (alone: the table path)
    again = compiler.compile_batch(big, 0)  # the dictionary is reset between batches
    assert [d.to_text() for d in again] == [d.to_text() for d in dems]
    assert compiler.compile(small, 1).hyperedges() == port.compile(small, 1)[0]


def test_pipelined_batch_matches_unpipelined():
    """GP_OPT_PIPELINE: a batch compiled as overlapped sub-batches (host
    packing || upload || device work || download) is bit-identical to the
    one-pass batch, including the global offsets of the flat batch view."""
    gens = [gp.gen_bb72_branch(b, rounds=3) for b in range(1100)]
    comp = gp.Compiler(0)
    comp.set_option(4, 0)
    want = [d.hyperedges() for d in comp.compile_batch(gens, 0)]
    comp.set_option(4, -1)
    for _ in range(2):  # the first call learns output sizes, the second is pipelined
        got = [d.hyperedges() for d in comp.compile_batch(gens, 0)]
        assert got == want


SHARD_CASES = [("surface_d5_r5", lambda: gp.gen_surface(5, 5, 1e-3)),
               ("bb72_branch7_r4", lambda: gp.gen_bb72_branch(7, rounds=4)),
               ("surface_d11_r11_si1000", lambda: gp.gen_surface(11, 11, 1e-3, gp.NOISE_MODEL_SI1000))]


@pytest.mark.parametrize("name,make", SHARD_CASES, ids=[n for n, _ in SHARD_CASES])
@pytest.mark.parametrize("level", [0, 2])
def test_fault_range_shards_merge_to_whole_compile(compiler, name, make, level):
    """the merge of n fault-range shards' partial tables (in any
    order) is the DEM of the whole circuit, byte for byte; the shards
    partition the nonempty sources."""
    g = make()
    want = compiler.compile(g, level).to_text()
    whole = compiler.compile_shard(g, 0, 1, level)
    assert compiler.merge_partials([whole]).to_text() == want
    for n in (2, 3, 8):
        parts = [compiler.compile_shard(g, k, n, level) for k in range(n)]
        assert sum(p.num_sources for p in parts) == whole.num_sources
        assert sum(len(p.rec_words) for p in parts) == len(whole.rec_words)
        assert compiler.merge_partials(parts).to_text() == want
        assert compiler.merge_partials(parts[::-1]).to_text() == want


def test_fault_range_shard_layers_and_errors(compiler):
    g = gp.gen_surface(3, 3, 1e-3)
    n = g.num_layers + 3  # more shards than layers: the extra shards are empty
    parts = [compiler.compile_shard(g, k, n) for k in range(n)]
    assert compiler.merge_partials(parts).to_text() == compiler.compile(g, 0).to_text()
    assert any(p.num_sources == 0 for p in parts)
    with pytest.raises(ValueError, match="shard index"):
        compiler.compile_shard(g, 2, 2)
    other = compiler.compile_shard(gp.gen_surface(5, 2, 1e-3), 0, 1)
    with pytest.raises(ValueError, match="different circuits"):
        compiler.merge_partials([parts[0], other])
    assert compiler.merge_partials([parts[0].__class__(g.num_detectors, g.num_observables, np.zeros(0),
                                                       np.zeros(1, np.uint32), np.zeros(0, np.uint32),
                                                       np.zeros(0, np.uint64))]).num_edges == 0


def test_fault_range_shards_device_tables(compiler):
    """GP_MEM_DEVICE partial tables (torch views of the workspace, cloned as
    an NCCL gather would) merge like host ones, alone or mixed with them."""
    import torch
    g = gp.gen_surface(7, 7, 1e-3, gp.NOISE_MODEL_SI1000)
    want = compiler.compile(g, 1).to_text()
    dev, host = [], []
    for k in range(4):
        t = compiler.compile_shard(g, k, 4, 1, on_device=True)
        dev.append(gp.DevicePartialTable(t.num_detectors, t.num_observables,
                                         *(x.clone() for x in t.arrays().values())))
        h = compiler.compile_shard(g, k, 4, 1)
        # same entries (sources in order; a source's records in emission order)
        assert np.array_equal(dev[-1].probs.cpu().numpy(), h.probs)
        assert np.array_equal(dev[-1].rec_offsets.cpu().numpy().view(np.uint32), h.rec_offsets)
        dw, db = dev[-1].rec_words.cpu().numpy().view(np.uint32), dev[-1].rec_bits.cpu().numpy().view(np.uint64)
        o = np.lexsort((db, dw))
        p = np.lexsort((h.rec_bits, h.rec_words))
        assert np.array_equal(dw[o], h.rec_words[p]) and np.array_equal(db[o], h.rec_bits[p])
        host.append(h)
    assert compiler.merge_partials(dev).to_text() == want
    assert compiler.merge_partials([dev[0], host[1], dev[2], host[3]]).to_text() == want
    # a device view of this compiler's own workspace is consumed before reuse
    last = compiler.compile_shard(g, 3, 4, 1, on_device=True)
    assert compiler.merge_partials(host[:3] + [last]).to_text() == want
    assert torch.cuda.is_available()


def test_malformed_partial_table_rejected(compiler):
    g = gp.gen_surface(3, 2, 1e-3)
    t = compiler.compile_shard(g, 0, 1)
    bad = gp.PartialTable(t.num_detectors, t.num_observables, t.probs, t.rec_offsets,
                          t.rec_words + np.uint32(1000), t.rec_bits)
    with pytest.raises(ValueError, match="malformed partial table"):
        compiler.merge_partials([bad])
    assert compiler.merge_partials([t]).to_text() == compiler.compile(g, 0).to_text()


def test_compile_sharded_over_nccl_single_rank():
    """shard.compile_sharded end to end through torch.distributed/NCCL
    (world size 1 on the one GPU: device tables, all-gather, device merge)."""
    import socket
    import torch.distributed as td
    from paper_2604_16613_b200.shard import compile_sharded
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    td.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        comp = gp.Compiler(0)
        g = gp.gen_bb72_branch(5, rounds=4)
        assert compile_sharded(comp, g, 2).to_text() == comp.compile(g, 2).to_text()
    finally:
        td.destroy_process_group()


@pytest.mark.parametrize("level", [0, 1, 2])
def test_direct_batch_traversal_all_levels(compiler, port, level):
    """>= 2 x SMs circuits take the batch traversal (one CTA per circuit, all
    six words, source-major emission of every component kind); each DEM
    equals the single-circuit compile (the split walk path) and the oracle."""
    gens = [gp.gen_bb72_branch(b, rounds=2) for b in range(300)] + [gp.gen_surface(3, 2, 2e-3),
                                                                    gp.gen_bb72_branch(5)]  # W = 6: 6-word CTAs
    dems = compiler.compile_batch(gens, level)
    for i in (0, 1, 150, 299, 300, 301):
        assert dems[i].to_text() == compiler.compile(gens[i], level).to_text()
    assert dems[7].hyperedges() == port.compile(gens[7].to_circuit(), level)[0]


# ---------------------------------------------------------------- headline parity
BRANCHES = np.load(GOLDEN / "bb72_branches_r6_L0.npz")


def branch_views(first: int, count: int):
    gens = [gp.gen_bb72_branch(b) for b in range(first, first + count)]
    from paper_2604_16613_b200 import _native as N
    arr = (N.CircuitView * count)()
    for i, g in enumerate(gens):
        arr[i] = g.view()[0]
    return gens, arr


def check_branch_batch(comp, out, first, count):
    eoff = np.ctypeslib.as_array(out.edge_offsets, shape=(count + 1,))
    assert np.array_equal(np.diff(eoff), BRANCHES["edges"][first:first + count].astype(np.uint64))
    got = comp.batch_digests(out)
    bad = np.nonzero(got != BRANCHES["digests"][first:first + count])[0]
    assert bad.size == 0, f"{bad.size} branch DEMs differ from the reference (first: {first + int(bad[0])})"


@pytest.mark.parametrize("pipeline", [0, -1], ids=["one-pass", "pipelined"])
def test_headline_branch_batch_matches_reference(pipeline):
    """BASELINE config 5 exactly as bench.py runs it: 4,096 BB [[72,12,6]] r6
    branches at L0 in one gp_compile_batch call -- the batch traversal
    (traverse_kernel<6>, one CTA per circuit), one 4,096-circuit reduce
    (pipeline off: what gp_replay times) or the 3-lane pipelined sub-batches
    (the e2e path) -- every branch's DEM equal to the reference's (digest of
    ids + probability bits; tests/golden/bb72_branches_r6_L0.npz)."""
    gens, views = branch_views(0, 4096)
    comp = gp.Compiler(0)
    comp.set_option(4, pipeline)
    for _ in range(2 if pipeline else 1):  # (pipelined: the first call learns the output sizes)
        out, st = comp.compile_batch_raw(views, 0)
        check_branch_batch(comp, out, 0, 4096)
    # the replay (bench.py's `value`) re-runs the resident plan; the next compile is still exact
    comp.replay(2)
    out, _ = comp.compile_batch_raw(views, 0)
    check_branch_batch(comp, out, 0, 4096)


def test_pipelined_batch_one_lane_matches_reference(monkeypatch):
    """The pipelined batch with one compute lane (GP_PIPE_LANES=1: every
    sub-batch's kernels in one stream, its image and workspace reused in
    stream order) gives the reference DEMs of the headline branches."""
    monkeypatch.setenv("GP_PIPE_LANES", "1")
    gens, views = branch_views(0, 4096)
    comp = gp.Compiler(0)
    comp.set_option(4, -1)
    for _ in range(2):
        out, _ = comp.compile_batch_raw(views, 0)
        check_branch_batch(comp, out, 0, 4096)


def test_headline_branch_batch_rank1_range():
    """Branch ids 4096..8191 (rank 1's shard at N = 2), small item hint first:
    the items-capacity re-run at the bench's scale."""
    gens, views = branch_views(4096, 4096)
    comp = gp.Compiler(0)
    comp.set_option(4, 0)
    small, sv = branch_views(0, 300)
    comp.compile_batch_raw(sv, 0)  # learns small capacities
    out, _ = comp.compile_batch_raw(views, 0)
    check_branch_batch(comp, out, 4096, 4096)


def test_reference_adaptive_shots(ref):
    """The reference's own adaptive workload (run_adaptive_shot,
    adaptive.cpp:382-391: Iceberg-concatenated d = 4 shots) compiled as one
    GPU batch (>= 2 x SMs circuits: the batch traversal) and one by one; each
    DEM's text equals the DEM the reference compiled for that shot."""
    shots = [ref.adaptive_shot(4, 0, 0, 1e-3, 1, s) for s in range(400)]
    circuits = [gp.parse_circuit(h.text()) for h, _ in shots]
    dems = gp.Compiler(0).compile_batch(circuits, 0)
    for i, (d, (_, text)) in enumerate(zip(dems, shots)):
        assert d.to_text() == text, i
    comp = gp.Compiler(0)
    for i in (0, 7, 399):
        assert comp.compile(circuits[i], 0).to_text() == shots[i][1]


def test_reference_acceptance_gate_through_dropin():
    """The reference's acceptance gate (tests/acceptance.cpp, 10 criteria)
    linked WITHOUT compile.cpp: every compile_circuit call -- criteria 2, 5,
    6, 8, 10 and the adaptive shots of 7 and 8 -- goes through the drop-in
    demc::compile_circuit of libgreenpeas.so on the GPU (oracle/Makefile
    `dropin`)."""
    exe = ROOT / "oracle" / "_ref" / "demc_acceptance_gpu"
    if not exe.exists():
        pytest.skip("oracle/_ref/demc_acceptance_gpu not built (needs the reference sources)")
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900)
    lines = [x for x in out.stdout.splitlines() if x.startswith(("PASS", "FAIL"))]
    assert len(lines) == 10 and all(x.startswith("PASS") for x in lines), out.stdout + out.stderr
    assert out.returncode == 0


# ---------------------------------------------------------------- device branch generation

def test_device_generated_branches_match_reference():
    """gp_compile_bb_branches: the 4,096 headline branches generated on the
    GPU from (seed, branch id) -- no host circuits -- give every branch's
    reference DEM (digests of tests/golden/bb72_branches_r6_L0.npz); an offset
    range too (branch ids 3,000 .. 4,095), and repeated calls."""
    comp = gp.Compiler(0)
    spec = gp.bb72_branch_spec()
    for _ in range(2):
        out, st = comp.compile_bb_branches_raw(spec, 0, 4096, 0)
        check_branch_batch(comp, out, 0, 4096)
    assert st["h2d_bytes"] < 4096 * 512  # the image head only: no circuits cross PCIe
    out, _ = comp.compile_bb_branches_raw(spec, 3000, 1096, 0)
    check_branch_batch(comp, out, 3000, 1096)


def test_every_rank_range_of_the_scaling_run_matches_reference():
    """The N = 8 scaling run's whole workload: rank r compiles branch ids
    4,096 r .. 4,096 r + 4,095, so 32,768 branches in all -- every one of them
    generated on the device and compiled in rank-sized batches, each DEM equal
    to the reference's (the golden digests cover all 32,768); rank 7's range
    also from host circuits through the pipelined batch path."""
    comp = gp.Compiler(0)
    spec = gp.bb72_branch_spec()
    for first in range(0, 8 * 4096, 4096):
        out, _ = comp.compile_bb_branches_raw(spec, first, 4096, 0)
        check_branch_batch(comp, out, first, 4096)
    gens, views = branch_views(7 * 4096, 4096)
    comp.set_option(4, -1)
    for _ in range(2):
        out, _ = comp.compile_batch_raw(views, 0)
        check_branch_batch(comp, out, 7 * 4096, 4096)


@pytest.mark.parametrize("case", ["bb72-cp0.3-L2", "bb72-cp0.9-L1", "bb144-full-L0", "bb72-si1000-L0"])
def test_device_generated_branches_equal_host_generated(case):
    """Other specs (check probability, level, code, noise model): the device
    generator's batch DEM equals gp_compile_batch over gen_bb's host circuits
    (digest per circuit)."""
    kw = {"bb72-cp0.3-L2": dict(l=6, m=6, rounds=6, noise_model=0, check_prob=0.3, refresh=3, seed=7, level=2,
                                first=1000, count=300),
          "bb72-cp0.9-L1": dict(l=6, m=6, rounds=8, noise_model=2, check_prob=0.9, refresh=0, seed=3, level=1,
                                first=5, count=320),
          "bb144-full-L0": dict(l=12, m=6, rounds=3, noise_model=2, check_prob=1.0, refresh=0, seed=1, level=0,
                                first=0, count=4),
          "bb72-si1000-L0": dict(l=6, m=6, rounds=6, noise_model=1, check_prob=0.5, refresh=2, seed=11, level=0,
                                 first=77, count=400)}[case]
    level, first, count = kw.pop("level"), kw.pop("first"), kw.pop("count")
    l, m = kw.pop("l"), kw.pop("m")
    spec = gp.bb_spec(l, m, p=2e-3, **kw)
    comp = gp.Compiler(0)
    comp.set_option(4, 0)
    out, _ = comp.compile_bb_branches_raw(spec, first, count, level)
    got = comp.batch_digests(out)
    gens = [gp.gen_bb(l, m, p=2e-3, branch=b, **kw) for b in range(first, first + count)]
    from paper_2604_16613_b200 import _native as N
    arr = (N.CircuitView * count)()
    for i, g in enumerate(gens):
        arr[i] = g.view()[0]
    ref_comp = gp.Compiler(0)
    ref_comp.set_option(4, 0)
    want_out, _ = ref_comp.compile_batch_raw(arr, level)
    want = ref_comp.batch_digests(want_out)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{bad.size} of {count} differ (first: branch {first + int(bad[0])})"


def test_device_generated_branches_errors():
    comp = gp.Compiler(0)
    with pytest.raises(ValueError, match="branch count"):
        comp.compile_bb_branches_raw(gp.bb72_branch_spec(), 0, 0, 0)
    with pytest.raises(ValueError, match="l, m >= 2"):
        comp.compile_bb_branches_raw(gp.bb_spec(1, 6), 0, 4, 0)
    with pytest.raises(ValueError, match="correlation level"):
        comp.compile_bb_branches_raw(gp.bb72_branch_spec(), 0, 4, 3)


# ---------------------------------------------------------------- two real ranks on the one GPU

def _two_proc_worker(rank, world, port, q):
    import os
    import sys
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, str(ROOT))
    try:
        import numpy as np
        import torch.distributed as td

        import bench
        import paper_2604_16613_b200 as gp
        from paper_2604_16613_b200 import shard
        td.init_process_group("gloo")
        comp = gp.Compiler(0)
        res = {}
        # fault-range sharding of one circuit, fold spread over the owners, DEM gathered to rank 0
        for name, make, level in (("d11_si1000", lambda: gp.gen_surface(11, 11, 1e-3, gp.NOISE_MODEL_SI1000), 0),
                                  ("bb144", lambda: gp.gen_bb144(6), 2)):
            g = make()
            tm = {}
            dem = shard.compile_sharded(comp, g, level, timings=tm)
            res[name] = (None if dem is None else dem.to_text() == comp.compile(g, level).to_text(),
                         tm["merged_entries"])
        # branch batches sharded by branch id, DEM tables gathered to rank 0
        per = 300
        circuits = bench.build_branches(rank * per, per)
        views = bench.views_of(circuits)
        out, _ = comp.compile_batch_raw(views, 0)
        z = np.load(bench.GOLDEN_BRANCHES)
        ok = bool(np.array_equal(comp.batch_digests(out), z["digests"][rank * per:(rank + 1) * per]))
        from paper_2604_16613_b200 import _native as N
        E = int(out.num_edges)
        got = shard.gather_to_root({"probs": N.copy_f64(out.probs, E),
                                    "edge_offsets": N.copy_u64(out.edge_offsets, per + 1)}, "cpu", 0)
        res["branches"] = (ok, None if got is None else [len(x) for x in got["probs"]],
                           None if got is None else [int(x[-1]) for x in got["edge_offsets"]])
        td.destroy_process_group()
        q.put((rank, res))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, "error " + traceback.format_exc()))


def test_two_process_sharded_compile_and_gather():
    """SURVEY 8e with two real ranks (two processes, gloo, both on cuda:0):
    compile_sharded of one circuit -- shard compiles, all-to-all of the
    entries to their owners, each owner's device merge (the fold spread over
    ranks), owners' DEMs gathered to rank 0 -- is byte-identical to the
    one-process compile; branch-sharded batches match the reference digests
    and their DEM tables reach rank 0."""
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_two_proc_worker, args=(r, 2, port, q)) for r in range(2)]
    [p.start() for p in procs]
    res = dict(q.get(timeout=600) for _ in procs)
    [p.join(timeout=120) for p in procs]
    for r in (0, 1):
        assert not isinstance(res[r], str), res[r]
    for name in ("d11_si1000", "bb144"):
        assert res[0][name][0] is True, name
        assert res[1][name][0] is None
        assert res[0][name][1] > 0 and res[1][name][1] > 0  # both owners folded a share
    assert res[0]["branches"][0] and res[1]["branches"][0]
    assert res[1]["branches"][1] is None
    assert res[0]["branches"][2][0] > 0 and res[0]["branches"][2][1] > 0


# ---------------------------------------------------------------- one-CTA tiny compiles

@pytest.mark.parametrize("fx", FIXTURES, ids=lambda p: p.name)
def test_tiny_and_general_paths_agree_on_fixtures(fx, monkeypatch):
    """Single circuits with D + O <= 64 compile in one CTA (gp_tiny.cuh);
    the general multi-kernel pipeline (GP_NO_TINY) gives the same bytes, and
    both equal the reference's golden text."""
    circuit, level, text, golden = fixture_case(fx)
    comp = gp.Compiler(0)
    assert comp.compile(circuit, level).to_text() == text
    monkeypatch.setenv("GP_NO_TINY", "1")
    assert gp.Compiler(0).compile(circuit, level).to_text() == text


@pytest.mark.parametrize("level", [0, 1, 2])
def test_tiny_path_random_small_circuits(port, level, monkeypatch):
    """Surface / repetition circuits that fit one word, every level: the
    one-CTA path equals the oracle and the general pipeline; the launch count
    shows the one kernel."""
    cases = [gp.gen_surface(3, 3, 1e-3), gp.gen_surface(3, 5, 2e-3, gp.NOISE_MODEL_SI1000), gp.gen_repetition(5, 4, 1e-2),
             gp.gen_surface(3, 1, 1e-3)]
    comp = gp.Compiler(0)
    for i, g in enumerate(cases):
        dem = comp.compile(g, level)
        if i == 0:  # (d3 r3 fits at every level; larger ones may exceed the one-CTA shared memory)
            assert comp.last_stats["kernel_launches"] == 1
        assert dem.hyperedges() == port.compile(g.to_circuit(), level)[0]
        monkeypatch.setenv("GP_NO_TINY", "1")
        assert gp.Compiler(0).compile(g, level).to_text() == dem.to_text()
        monkeypatch.delenv("GP_NO_TINY")


# ---------------------------------------------------------------- circuits too wide for on-chip walk state

@pytest.mark.parametrize("name,level", [("surface_d11_r11_si1000", 1), ("bb144_r12_uniform", 2),
                                        ("surface_d25_r25_paper", 0)])
def test_global_state_walk_matches_reference(name, level, monkeypatch):
    """walk_wide_kernel (the walk state in global memory, the fallback for
    circuits beyond ~4,800 qubits) forced on the BASELINE circuits: the DEM
    hashes equal the reference's (tests/golden/full_size.json)."""
    monkeypatch.setenv("GP_WALK_WIDE", "1")
    g = FULL_MAKERS[name]()
    comp = gp.Compiler(0)
    dem = comp.compile(g, level)
    assert sha(dem.to_text()) == FULL[name]["levels"][str(level)]["dem_sha256"]


def test_circuit_wider_than_shared_memory(ref):
    """Surface d = 51, 2 rounds: 5,201 qubits, beyond the on-chip walk state
    (round 1 failed with "circuit too wide"); compiled through the global-state
    walk, its DEM text equals the reference's."""
    g = gp.gen_surface(51, 2, 1e-3)
    assert g.num_qubits > 5000
    got = gp.Compiler(0).compile(g, 0).to_text()
    want, _ = ref.parse(g.to_text()).compile(0)
    assert got == want


def test_signature_spanning_many_words(ref):
    """A measurement flip whose signature has detectors in 18 different
    64-bit words (more than round 1's 16-record limit): the record slots grow
    on overflow and the DEM text equals the reference's."""
    n = 1100
    lines = [f"M(0.01) {' '.join(str(q) for q in range(n))}", "X_ERROR(0.02) 0 5 70"]
    # detector d holds measurement d, and measurement 0 when d is a multiple of 64
    for d in range(n):
        recs = {n - d}
        if d % 64 == 0 and d:
            recs.add(n)
        lines.append("DETECTOR " + " ".join(f"rec[-{k}]" for k in sorted(recs)))
    text = "\n".join(lines) + "\n"
    want, _ = ref.parse(text).compile(0)
    comp = gp.Compiler(0)
    assert comp.compile(gp.parse_circuit(text), 0).to_text() == want


# ---------------------------------------------------------------- drop-in under concurrent callers
def _shim_pool_digests(views, levels, threads):
    import ctypes as C
    from paper_2604_16613_b200 import _native as N
    L = C.CDLL(str(N.LIB_PATH.parent / "libgp_shimbench.so"))
    n = len(levels)
    lv = np.asarray(levels, np.uint8)
    dig = np.zeros(n, np.uint64)
    st = np.full(n, -1, np.int32)
    msg = C.create_string_buffer(128 * n)
    L.sb_shim_pool_digests.restype = C.c_int
    L.sb_shim_pool_digests(views, C.c_uint32(n), lv.ctypes.data_as(C.c_void_p), C.c_uint32(threads),
                           dig.ctypes.data_as(C.c_void_p), st.ctypes.data_as(C.c_void_p), msg)
    msgs = [msg.raw[i * 128:(i + 1) * 128].split(b"\0")[0].decode() for i in range(n)]
    return dig, st, msgs


def test_dropin_concurrent_callers_match_reference():
    """Reentrancy at scale, the demc_main.cpp:184-195 pattern: 16 host threads
    calling demc::compile_circuit at once (one GPU context each, one shared
    packing pool): every branch DEM equals the reference's."""
    gens, views = branch_views(0, 1024)
    dig, st, _ = _shim_pool_digests(views, [0] * 1024, 16)
    assert (st == 0).all()
    bad = np.nonzero(dig != BRANCHES["digests"][:1024])[0]
    assert bad.size == 0, f"{bad.size} DEMs differ (first: {int(bad[0])})"


def test_dropin_concurrent_mixed_levels_and_invalid_circuits():
    """Concurrent drop-in calls of different levels, with invalid circuits among
    them: each invalid one raises its own invalid_argument with the
    reference's message, the others are exact."""
    from paper_2604_16613_b200 import _native as N
    n = 192
    gens = [gp.gen_bb72_branch(b) for b in range(n)]
    levels = [2 if i % 5 == 0 else 0 for i in range(n)]
    keep, arr = [], (N.CircuitView * n)()
    for i, g in enumerate(gens):
        c = g.to_circuit()
        if i % 37 == 3:
            c = gp.Circuit(**{**c.__dict__, "det_meas": c.det_meas + 100000})
        v, a = N.view_of(c)
        keep.append(a)
        arr[i] = v
    dig, st, msgs = _shim_pool_digests(arr, levels, 16)
    comp = gp.Compiler(0)
    l2 = [i for i in range(n) if levels[i] == 2 and i % 37 != 3]
    sub = (N.CircuitView * len(l2))(*[arr[i] for i in l2])
    out, _ = comp.compile_batch_raw(sub, 2)
    want_l2 = dict(zip(l2, comp.batch_digests(out)))
    for i in range(n):
        if i % 37 == 3:
            assert st[i] == 1 and msgs[i] == "detector references a measurement without a leaf", (i, st[i], msgs[i])
        elif levels[i] == 2:
            assert st[i] == 0 and dig[i] == want_l2[i], i
        else:
            assert st[i] == 0 and dig[i] == BRANCHES["digests"][i], i

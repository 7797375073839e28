"""CPU: the headline-workload goldens (tests/golden/bb72_branches_r6_L0.npz)
and the DEM digest both sides use.

The npz holds, for every BB [[72,12,6]] r6 L0 branch circuit bench.py
compiles at N = 1..8 (branch ids 0 .. 8*4096-1), the reference's hyperedge
count and DEM digest (gp_dem_digest's definition, restated over demc::Dem in
oracle/ref_capi.cpp). These tests pin that file to the reference itself (a
random sample recompiled by oracle/_ref), the repo's generator to the
circuits the reference compiled, and the two digest implementations to each
other. The GPU side of the comparison is tests/test_gpu.py."""

import hashlib

import numpy as np
import pytest

import paper_2604_16613_b200 as gp
from oracle.bindings import parse_dem_text

from .conftest import FIXTURES, GOLDEN

BRANCHES = np.load(GOLDEN / "bb72_branches_r6_L0.npz")


def dem_of(edges, nd, no):
    doff, dids, ooff, oids, probs = [0], [], [0], [], []
    for d, o, p in edges:
        dids += d
        oids += o
        doff.append(len(dids))
        ooff.append(len(oids))
        probs.append(p)
    return gp.Dem(nd, no, np.array(doff, np.uint64), np.array(dids, np.uint32), np.array(ooff, np.uint64),
                  np.array(oids, np.uint32), np.array(probs, np.float64))


def test_golden_file_shape():
    assert BRANCHES["edges"].shape == (8 * 4096,) and BRANCHES["digests"].shape == (8 * 4096,)
    assert int(BRANCHES["seed"]) == 1 and int(BRANCHES["rounds"]) == 6 and int(BRANCHES["level"]) == 0
    # every branch's DEM is distinct (no circuit-level dedup available at p = 1e-3, check_prob = 1/2)
    assert len(np.unique(BRANCHES["digests"])) == 8 * 4096


def test_generator_matches_golden_circuits():
    h = hashlib.sha256()
    for b in range(256):
        h.update(gp.gen_bb72_branch(b).to_text().encode())
    assert h.digest() == bytes(BRANCHES["circuits_0_255_sha256"])


def test_reference_reproduces_golden_sample(ref):
    """A random sample of branches recompiled by the reference library now."""
    rng = np.random.default_rng(11)
    ids = sorted(set(rng.integers(0, 8 * 4096, 40).tolist()) | {0, 4095, 4096, 8 * 4096 - 1})
    for b in ids:
        (c,) = ref.gen_bb72_branches(b, 1)
        e, d = ref.compile_digests([c], 0)
        assert int(e[0]) == int(BRANCHES["edges"][b]) and int(d[0]) == int(BRANCHES["digests"][b]), b


def test_reference_branch_text_is_the_repo_generator(ref):
    for b in (0, 17, 4095, 30000):
        (c,) = ref.gen_bb72_branches(b, 1)
        assert c.text() == gp.gen_bb72_branch(b).to_text()


@pytest.mark.parametrize("fx", FIXTURES, ids=lambda p: p.name)
def test_digest_agrees_with_reference_restatement(ref, fx):
    text = (fx / "expected.dem").read_text()
    c = gp.parse_circuit((fx / "circuit.txt").read_text())
    d = dem_of(parse_dem_text(text), c.num_detectors, c.num_observables)
    assert d.digest() == ref.dem_text_digest(text, c.num_detectors, c.num_observables)


def test_digest_sees_every_field():
    base = dem_of([((0, 1), (), 0.125), ((1,), (0,), 0.0625)], 2, 1)
    variants = [dem_of([((0, 1), (), 0.125), ((1,), (0,), 0.0625000000000001)], 2, 1),
                dem_of([((0, 1), (), 0.125), ((1,), (), 0.0625)], 2, 1),
                dem_of([((0,), (1,), 0.125), ((1,), (0,), 0.0625)], 2, 2),
                dem_of([((0, 1), (), 0.125)], 2, 1),
                dem_of([((0, 1), (), 0.125), ((1,), (0,), 0.0625)], 3, 1)]
    assert len({base.digest(), *(v.digest() for v in variants)}) == 1 + len(variants)

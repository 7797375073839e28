"""CPU: pins the plain-C restatement oracle (oracle/demc_oracle.c) against the
reference's golden fixtures, known-answer tests and the reference library
itself, so that it can serve as the checker of the GPU path."""

import math
import random

import numpy as np
import pytest

import paper_2604_16613_b200 as gp
from oracle.bindings import parse_dem_text

from .conftest import FIXTURES, GOLDEN, fixture_case


@pytest.mark.parametrize("fx", FIXTURES, ids=lambda p: p.name)
def test_port_matches_golden_fixture(port, fx):
    """test_frame.cpp:96-120: oracle == frozen goldens, bit-exact probabilities."""
    circuit, level, _, golden = fixture_case(fx)
    edges, _, _ = port.compile(circuit, level)
    assert edges == golden


@pytest.mark.parametrize("fx", FIXTURES, ids=lambda p: p.name)
def test_forward_oracle_matches_golden_fixture(port, fx):
    circuit, level, _, golden = fixture_case(fx)
    edges, _, _ = port.forward(circuit, level)
    assert edges == golden


def test_criterion1_handwritten_classes(port):
    """acceptance.cpp:70-104: 26 placements, 9 classes, {3,8,13} merged, 12 -> {D2,D3}."""
    circuit, level, _, _ = fixture_case(GOLDEN / "fixtures" / "rep_handwritten")
    edges, members, S = port.compile(circuit, level)
    assert circuit.num_detectors == 4 and S == 26 and len(edges) == 9
    for e, mem in zip(edges, members):
        if 3 in mem:
            assert sorted(mem) == [3, 8, 13]
        if 12 in mem:
            assert e[0] == (2, 3)


def test_fnv1_known_answers(port):
    """test_dem.cpp:23-31."""
    assert port.fnv1_64([]) == 0xCBF29CE484222325
    assert port.fnv1_64([1]) == 0xE3757CA7D64666EA
    assert port.fnv1_64([1, 0]) != port.fnv1_64([1])


def test_merge_prob_known_answers(port):
    """test_dem.cpp:34-36, acceptance.cpp:131-146."""
    assert math.isclose(port.merge_prob(0.1, 0.2), 0.26, rel_tol=1e-15)
    assert port.merge_prob(0.3, 0.0) == 0.3
    assert port.merge_prob(0.5, 0.37) == 0.5
    rng = random.Random(1234)
    for _ in range(2000):
        a, b, c = rng.random(), rng.random(), rng.random()
        assert port.merge_prob(a, b) == gp.merge_prob(a, b)
        assert abs(port.merge_prob(a, b) - port.merge_prob(b, a)) <= 1e-15
        m1 = port.merge_prob(port.merge_prob(a, b), c)
        m2 = port.merge_prob(a, port.merge_prob(b, c))
        assert abs(m1 - m2) <= 1e-15


def test_fold_known_answers():
    """test_dem.cpp:54-68 / 112-122: sorted fold from 0."""
    p = 0.0
    for _ in range(3):
        p = gp.merge_prob(p, 0.01)
    assert math.isclose(p, 0.029404, rel_tol=1e-15)
    p = 0.0
    for _ in range(7):
        p = gp.merge_prob(p, 0.01)
    assert math.isclose(p, 0.06593723337664, rel_tol=1e-15)


@pytest.mark.parametrize("name", ["rep_d3_r2", "rep_d5_r3", "surface_d3_r3", "surface_d4_r2",
                                  "surface_d5_r5_si1000", "surface_d5_r3_onlyz"])
@pytest.mark.parametrize("level", [0, 1, 2])
def test_port_matches_reference_generated_goldens(port, name, level):
    """The committed reference outputs (tests/golden/make_goldens.py)."""
    d = GOLDEN / "generated"
    circuit = gp.parse_circuit((d / f"{name}.circuit.txt").read_text())
    golden = parse_dem_text((d / f"{name}.L{level}.dem").read_text())
    edges, _, _ = port.compile(circuit, level)
    assert edges == golden


@pytest.mark.parametrize("d,r", [(3, 2), (3, 3)])
@pytest.mark.parametrize("level", [0, 1, 2])
def test_criterion2_port_vs_forward(port, d, r, level):
    """acceptance.cpp:107-127: pipeline == forward oracle across codes and levels."""
    c = gp.gen_surface(d, r, 1e-3).to_circuit()
    a, _, _ = port.compile(c, level)
    b, _, _ = port.forward(c, level)
    assert a == b


def test_port_matches_live_reference(port, ref):
    """Restatement vs the reference library on circuits outside the corpus."""
    for g in (gp.gen_bb(6, 6, rounds=2, p=1e-3), gp.gen_bb72_branch(11, rounds=4),
              gp.gen_surface(7, 3, 2e-3, gp.NOISE_MODEL_SI1000)):
        text = g.to_text()
        c = gp.parse_circuit(text)
        rc = ref.parse(text)
        for level in (0, 1, 2):
            dem, _ = rc.compile(level)
            edges, _, _ = port.compile(c, level)
            assert edges == parse_dem_text(dem)


def test_level_monotone_counts(port):
    """acceptance.cpp:160-179."""
    for g in (gp.gen_repetition(5, 3, 2e-3), gp.gen_surface(4, 2, 1e-3)):
        c = g.to_circuit()
        n = [len(port.compile(c, lv)[0]) for lv in (0, 1, 2)]
        assert n[0] <= n[1] <= n[2]


def test_oracle_errors(port):
    """eec.cpp:44-46: init_leaves rejects detectors on missing measurements."""
    c = gp.parse_circuit("M 0\nDETECTOR rec[-1]\n")
    c.det_meas = np.array([5], np.uint32)
    with pytest.raises(ValueError, match="detector references a measurement without a leaf"):
        port.compile(c, 0)

"""CPU: circuit grammar, generators (pinned against the reference
generators) and the workload circuits' noiseless soundness."""

import numpy as np
import pytest

import paper_2604_16613_b200 as gp

from .conftest import FIXTURES


def test_parse_rec_resolution():
    c = gp.parse_circuit("M 0\nM 1\nDETECTOR rec[-2] rec[-1]\nOBSERVABLE_INCLUDE(0) rec[-1]\n")
    assert c.num_measurements == 2 and c.num_layers == 1
    assert list(c.det_meas) == [0, 1] and list(c.obs_meas) == [1]


@pytest.mark.parametrize("text,msg", [
    ("CX 0 0\n", "CX control equals target"),
    ("M 0\nDETECTOR rec[-2]\n", "reaches before the first measurement"),
    ("FOO 1\n", "unsupported instruction"),
    ("X_ERROR 0\n", "needs a probability argument"),
    ("M 0\nDETECTOR rec[-1] rec[-1]\n", "cancels to empty"),
])
def test_parse_errors(text, msg):
    with pytest.raises(ValueError, match=msg):
        gp.parse_circuit(text)


def test_validate_rejects_conflicts():
    with pytest.raises(ValueError, match="used by two gates"):
        gp.parse_circuit("H 0\nCX 0 1\n")
    with pytest.raises(ValueError, match="DEPOLARIZE2 targets"):
        gp.parse_circuit("CX 0 1\nH 2\nDEPOLARIZE2(0.1) 0 2\n")


@pytest.mark.parametrize("fx", FIXTURES, ids=lambda p: p.name)
def test_serialize_round_trip(fx):
    c = gp.parse_circuit((fx / "circuit.txt").read_text())
    assert gp.parse_circuit(gp.serialize_circuit(c)).same_as(c)


@pytest.mark.parametrize("d,r,p", [(3, 3, 1e-3), (5, 2, 2e-3), (11, 11, 1e-3)])
def test_surface_generator_matches_reference(ref, d, r, p):
    """gp_gen_surface reproduces gen_surface (codes.cpp:245-333) exactly."""
    mine = gp.gen_surface(d, r, p).to_circuit()
    theirs = gp.parse_circuit(ref.gen_surface(d, r, p).text())
    assert mine.same_as(theirs)


def test_repetition_generator_matches_reference(ref):
    mine = gp.gen_repetition(5, 3, 2e-3).to_circuit()
    theirs = gp.parse_circuit(ref.gen_repetition(5, 3, 2e-3).text())
    assert mine.same_as(theirs)


def test_generated_text_parses_back():
    for g in (gp.gen_bb(6, 6, rounds=2), gp.gen_surface(5, 3, 1e-3, gp.NOISE_MODEL_SI1000),
              gp.gen_bb72_branch(2, rounds=4)):
        assert gp.parse_circuit(g.to_text()).same_as(g.to_circuit())


@pytest.mark.parametrize("name,make", [
    ("bb72", lambda: gp.gen_bb(6, 6, rounds=3, p=0.0)),
    ("bb144", lambda: gp.gen_bb(12, 6, rounds=2, p=0.0)),
    ("bb72_branch", lambda: gp.gen_bb(6, 6, rounds=6, p=0.0, noise_model=0, check_prob=0.5, refresh=3, branch=9)),
    ("si1000", lambda: gp.gen_surface(5, 3, 0.0, gp.NOISE_MODEL_SI1000)),
])
def test_noiseless_detectors_are_deterministic(ref, name, make):
    """acceptance.cpp:203-232 on the new generators: with collapse
    randomisation on, a noiseless circuit never fires a detector
    (sample_detector_values, frame.cpp:241-248, run by the reference)."""
    assert ref.parse(make().to_text()).sample_fired(7, 100) == 0


def test_bb_code_parameters():
    g = gp.gen_bb144(12, 1e-3)
    assert (g.num_qubits, g.num_observables) == (288, 12)
    assert g.num_detectors == 12 * 144  # 72 Z per round + 72 X from round 2 + 72 final
    b = gp.gen_bb72_branch(0)
    assert (b.num_qubits, b.num_observables) == (144, 12)


def test_branches_are_distinct():
    texts = {gp.gen_bb72_branch(b).to_text() for b in range(16)}
    assert len(texts) == 16


def test_logical_observables_are_deterministic(ref):
    """The 12 BB logical-Z observables must be deterministic in a noiseless
    Z-memory run: turn every OBSERVABLE_INCLUDE into a DETECTOR and let the
    reference's randomised-collapse sampler check it never fires."""
    import re
    for g in (gp.gen_bb(6, 6, rounds=2, p=0.0), gp.gen_bb(12, 6, rounds=1, p=0.0)):
        text = re.sub(r"OBSERVABLE_INCLUDE\(\d+\)", "DETECTOR", g.to_text())
        assert text.count("DETECTOR") >= 12
        assert ref.parse(text).sample_fired(3, 50) == 0

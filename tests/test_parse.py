"""The native circuit parser (gp_parse_circuit) against
the reference's own parse_circuit + validate_layers (circuit.cpp:107-326,
oracle/_ref): the same circuit -- compared through the reference serializer
(circuit.cpp:328-388) -- and, on malformed text, the same error message.
Large texts take the parallel chunked path (host pool); the error corpus
also runs through it (errors re-parse serially for the exact first error)."""
import pytest

import paper_2604_16613_b200 as gp

from .conftest import FIXTURES


def _ref():
    from oracle.bindings import REF_SO, RefLib
    if not REF_SO.exists():
        pytest.skip("oracle/_ref/libdemc_ref.so not built (reference sources absent)")
    return RefLib()


def _ref_result(ref, text):
    try:
        return "ok", ref.parse(text).text()
    except ValueError as e:
        return "err", str(e)


def _native_result(text):
    try:
        return "ok", gp.parse_circuit_native(text).to_text()
    except gp.CircuitParseError as e:
        return "err", str(e)


def _texts():
    out = [(fx.name, (fx / "circuit.txt").read_text()) for fx in FIXTURES]
    out += [("surface_d5_r4", gp.gen_surface(5, 4, 1e-3).to_text()),
            ("rep_d7_r3", gp.gen_repetition(7, 3, 2e-3).to_text()),
            ("bb72_branch3", gp.gen_bb72_branch(3).to_text()),
            ("surface_d3_si1000", gp.gen_surface(3, 3, 1e-3, gp.NOISE_MODEL_SI1000).to_text())]
    return out


@pytest.mark.parametrize("name,text", _texts(), ids=[n for n, _ in _texts()])
def test_native_parse_matches_reference(name, text):
    ref = _ref()
    assert _native_result(text) == _ref_result(ref, text)


def test_native_parse_large_text_parallel():
    """Megabytes of text (surface d15 r15: the chunked parallel path) parse to
    the reference's circuit; so does the same text with comments, blank lines,
    CRLF endings and tab separators."""
    ref = _ref()
    text = gp.gen_surface(15, 15, 1e-3).to_text()
    assert len(text) > (1 << 20)
    assert _native_result(text) == _ref_result(ref, text)
    noisy = "# header\n\n" + text.replace("\n", "  # c\r\n").replace(" ", "\t", 3)
    assert _native_result(noisy) == _ref_result(ref, noisy)


GOOD = "R 0 1 2\nTICK\nCX 0 1\nDEPOLARIZE2(0.01) 0 1\nTICK\nM(0.002) 0 1 2\nDETECTOR rec[-1] rec[-2]\n" \
       "OBSERVABLE_INCLUDE(0) rec[-3]\n"
BAD = {
    "unterminated": "H(0.1 0\n",
    "bad_number": "X_ERROR(0.1x) 0\n",
    "tick_targets": "TICK 3\n",
    "h_arg": "H(0.5) 0\n",
    "h_empty": "R\n",
    "cx_odd": "CX 0 1 2\n",
    "cx_same": "CX 1 1\n",
    "m_empty": "MR\n",
    "noise_noarg": "DEPOLARIZE1 0\n",
    "dep2_noarg": "DEPOLARIZE2 0 1\n",
    "dep2_odd": "DEPOLARIZE2(0.1) 0 1 2\n",
    "det_empty": "M 0\nDETECTOR\n",
    "det_cancel": "M 0\nDETECTOR rec[-1] rec[-1]\n",
    "det_before": "M 0\nDETECTOR rec[-2]\n",
    "det_zero": "M 0\nDETECTOR rec[-0]\n",
    "det_format": "M 0\nDETECTOR rec[1]\n",
    "det_range_then_format": "M 0\nDETECTOR rec[-3] rec[x]\n",
    "obs_noarg": "M 0\nOBSERVABLE_INCLUDE rec[-1]\n",
    "obs_frac": "M 0\nOBSERVABLE_INCLUDE(0.5) rec[-1]\n",
    "obs_dense": "M 0\nOBSERVABLE_INCLUDE(1) rec[-1]\n",
    "obs_dense_before_format": "M 0\nOBSERVABLE_INCLUDE(2) rec[x]\n",
    "unsupported": "Y 0\n",
    "qubit": "H a\n",
    "two_gates": "H 0\nCX 0 1\n",
    "flip_range": "M(1.5) 0\n",
    "noise_range": "X_ERROR(-0.1) 0\n",
    "dep2_pair": "CX 0 1\nDEPOLARIZE2(0.1) 1 0\n",
    "dep2_half_idle": "H 0\nDEPOLARIZE2(0.1) 0 2\n",
    "later_layer": "H 0\nTICK\nH 1 1\n",
    "empty_text": "",
    "comments_only": "# nothing\n\n   \n",
    "ticks_only": "TICK\nTICK\n",
}


@pytest.mark.parametrize("case", sorted(BAD))
def test_native_parse_errors_match_reference(case):
    ref = _ref()
    text = BAD[case]
    assert _native_result(text) == _ref_result(ref, text)


@pytest.mark.parametrize("case", sorted(BAD))
def test_native_parse_errors_in_large_text(case):
    """The same malformed line at the end of megabytes of valid text (the
    parallel pass fails, the serial re-parse reports the reference's first
    error with its line number)."""
    ref = _ref()
    big = gp.gen_surface(13, 13, 1e-3).to_text() + "TICK\n"
    text = big + BAD[case]
    assert _native_result(text) == _ref_result(ref, text)


def test_native_parse_good_small():
    ref = _ref()
    assert _native_result(GOOD) == _ref_result(ref, GOOD)


def test_cpp_dropin_parse_circuit(tmp_path):
    """demc::parse_circuit of the drop-in headers (include/demc/circuit.hpp)
    through libgreenpeas: a reference-style caller gets the circuit, a
    demc::ParseError with the line, or std::invalid_argument for layers."""
    import shutil
    import subprocess

    from .conftest import ROOT
    if shutil.which("g++") is None:
        pytest.skip("needs g++")
    src = tmp_path / "p.cpp"
    src.write_text(r'''
#include <cstdio>
#include "demc/circuit.hpp"
int main() {
    demc::Circuit c = demc::parse_circuit("R 0 1\nTICK\nCX 0 1\nTICK\nM(0.01) 0 1\nDETECTOR rec[-1] rec[-2]\n"
                                          "OBSERVABLE_INCLUDE(0) rec[-1]\n");
    std::printf("%u %zu %u %zu %zu %zu %.2f\n", c.num_qubits, c.layers.size(), c.num_measurements,
                c.detectors.size(), c.observables.size(), c.layers[2].annotations.size(),
                c.layers[2].gates[1].flip_prob);
    try { demc::parse_circuit("H 0\nCX 0 1 2\n"); } catch (const demc::ParseError &e) { std::printf("%zu|%s\n", e.line, e.what()); }
    try { demc::parse_circuit("H 0 0\n"); } catch (const std::invalid_argument &e) { std::printf("%s\n", e.what()); }
}
''')
    lib = ROOT / "paper_2604_16613_b200" / "_lib"
    exe = tmp_path / "p"
    subprocess.run(["g++", "-std=c++20", "-I", str(ROOT / "include"), str(src), str(lib / "libgreenpeas.so"),
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines()
    assert out == ["2 3 2 1 1 2 0.01", "2|line 2: CX needs an even number of targets",
                   "layer 0: qubit 0 used by two gates in one layer"]

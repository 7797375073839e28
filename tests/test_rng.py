"""gp_rng.h (the device branch generator's mt19937_64 / seed_seq /
uniform_real_distribution restatement) against the C++ standard library,
compiled for the host: 36,000 draws over edge-case seeds and branch ids."""
import shutil
import subprocess

import pytest

from .conftest import ROOT


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_rng_restatement_matches_std(tmp_path):
    exe = tmp_path / "rng_check"
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", str(ROOT / "paper_2604_16613_b200" / "csrc"),
                    str(ROOT / "tests" / "cpp" / "rng_check.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert out.stdout.strip() == "draws 36000 mismatches 0"

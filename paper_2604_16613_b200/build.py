"""In-tree build of libgreenpeas.so (sm_100a) -- no JIT cache, no pip install.

    python -m paper_2604_16613_b200.build            # build if stale
    python -m paper_2604_16613_b200.build --force

The shared library is written to paper_2604_16613_b200/_lib/ so it travels
with the repository snapshot to the GPU box. Host C++ is compiled by g++
(C++20, for std::to_chars), device code by nvcc for sm_100a only.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libgreenpeas.so"
# Benchmark harness of the C++ drop-in endpoint (bench.py only; links LIB).
SHIMBENCH = OUT_DIR / "libgp_shimbench.so"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = CUDA_HOME / "bin" / "nvcc"

CU_SOURCES = ["gp_kernels.cu"]
CPP_SOURCES = ["gp_api.cpp", "gp_pack.cpp", "gp_gen.cpp", "gp_parse.cpp", "demc_shim.cpp"]
HEADERS = ["gp_layout.h", "gp_device.h", "gp_pack.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd: list[str]) -> None:
    print(" ".join(str(c) for c in cmd), flush=True)
    subprocess.run([str(c) for c in cmd], check=True)


def _stale() -> bool:
    if not LIB.exists() or not SHIMBENCH.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in CU_SOURCES + CPP_SOURCES + HEADERS + ["gp_shimbench.cpp"]] + list(CSRC.glob("*.cuh"))
    deps += list((ROOT / "include").rglob("*.h*"))
    return any(p.stat().st_mtime > t for p in deps if p.exists())


def build(force: bool = False, verbose_ptxas: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    OUT_DIR.mkdir(exist_ok=True)
    objs = []
    inc = ["-I", str(ROOT / "include"), "-I", str(CSRC)]
    for src in CU_SOURCES:
        obj = OUT_DIR / (Path(src).stem + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "--expt-relaxed-constexpr", *inc, "-c", CSRC / src, "-o", obj]
        if verbose_ptxas:
            cmd[1:1] = ["-Xptxas", "-v"]
        _run(cmd)
        objs.append(obj)
    for src in CPP_SOURCES:
        obj = OUT_DIR / (Path(src).stem + ".o")
        _run(["g++", "-O2", "-std=c++20", "-fPIC", "-Wall", *inc, "-I", str(CUDA_HOME / "include"),
              "-c", CSRC / src, "-o", obj])
        objs.append(obj)
    tmp = LIB.with_suffix(".so.tmp")
    _run(["g++", "-shared", "-o", tmp, *objs, "-L", str(CUDA_HOME / "lib64"),
          "-lcudart_static", "-lpthread", "-ldl", "-lrt", "-Wl,--no-undefined"])
    os.replace(tmp, LIB)
    _run(["g++", "-O2", "-std=c++20", "-fPIC", "-shared", "-Wall", *inc, CSRC / "gp_shimbench.cpp", LIB,
          "-Wl,-rpath,$ORIGIN", "-lpthread", "-o", SHIMBENCH])
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)

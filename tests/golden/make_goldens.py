"""Regenerates the committed golden vectors from the REFERENCE implementation.

Run in the build container (needs /root/reference and oracle/_ref):

    make -C oracle ref && python tests/golden/make_goldens.py

For every workload circuit (produced by this repo's generators, whose output
is pinned against the reference generators where those exist) the reference
`demc::compile_circuit` (built from /root/reference sources by oracle/Makefile)
is run and its serialize_dem text is recorded:

* small cases: full text under tests/golden/generated/<case>.dem (+ circuit)
* BASELINE.json configs at full size: sha256 + hyperedge count in
  tests/golden/full_size.json, so the GPU path can be checked byte-for-byte
  at the sizes it is benchmarked on without shipping megabytes of text.
* the headline workload (config 5): every BB [[72,12,6]] r6 L0 branch
  circuit b = 0 .. 8 * 4096 - 1 (what bench.py compiles at N = 1..8), its
  hyperedge count and DEM digest (gp_dem_digest's definition, restated over
  the reference's demc::Dem in oracle/ref_capi.cpp) in
  tests/golden/bb72_branches_r6_L0.npz; plus a sha256 over the circuit text
  of branches 0..255 to tell generator drift from compiler drift.

    python tests/golden/make_goldens.py [small] [full] [branches]
"""

from __future__ import annotations

import hashlib
import json
import sys
import time

import numpy as np
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import paper_2604_16613_b200 as gp  # noqa: E402
from oracle.bindings import RefLib  # noqa: E402

OUT = Path(__file__).resolve().parent
SMALL = {
    "rep_d3_r2": lambda: gp.gen_repetition(3, 2, 1e-3),
    "rep_d5_r3": lambda: gp.gen_repetition(5, 3, 2e-3),
    "surface_d3_r3": lambda: gp.gen_surface(3, 3, 1e-3),
    "surface_d4_r2": lambda: gp.gen_surface(4, 2, 1e-3),
    "surface_d5_r5_si1000": lambda: gp.gen_surface(5, 5, 1e-3, gp.NOISE_MODEL_SI1000),
    "surface_d5_r3_onlyz": lambda: gp.gen_surface(5, 3, 1e-3, gp.NOISE_MODEL_PAPER, True),
}

FULL = {
    "bb72_r2_uniform": (lambda: gp.gen_bb(6, 6, rounds=2, p=1e-3), (0, 1, 2)),
    "bb72_branch3_r4": (lambda: gp.gen_bb72_branch(3, rounds=4), (0, 1, 2)),
    "surface_d3_r3_paper": (lambda: gp.gen_surface(3, 3, 1e-3), (0, 1, 2)),
    "surface_d11_r11_si1000": (lambda: gp.gen_surface(11, 11, 1e-3, gp.NOISE_MODEL_SI1000), (0, 1, 2)),
    "bb144_r12_uniform": (lambda: gp.gen_bb144(12, 1e-3), (0, 1, 2)),
    "surface_d25_r25_paper": (lambda: gp.gen_surface(25, 25, 1e-3), (0,)),
}
BRANCHES = 32


def sha(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()


BRANCH_TOTAL = 8 * 4096


def make_branch_goldens(ref) -> None:
    t0 = time.time()
    edges, digests = [], []
    chunk = 2048
    for first in range(0, BRANCH_TOTAL, chunk):
        hs = ref.gen_bb72_branches(first, chunk)
        e, d = ref.compile_digests(hs, 0)
        edges.append(e.astype(np.uint32))
        digests.append(d)
        print("branches", first + chunk, f"{time.time() - t0:.0f}s", flush=True)
    h = hashlib.sha256()
    for c in ref.gen_bb72_branches(0, 256):
        h.update(c.text().encode())
    np.savez_compressed(OUT / "bb72_branches_r6_L0.npz", edges=np.concatenate(edges),
                        digests=np.concatenate(digests),
                        circuits_0_255_sha256=np.frombuffer(bytes.fromhex(h.hexdigest()), np.uint8),
                        seed=np.uint64(1), rounds=np.uint32(6), level=np.uint32(0))


def main() -> None:
    parts = set(sys.argv[1:]) or {"small", "full", "branches"}
    ref = RefLib()
    if "branches" in parts:
        make_branch_goldens(ref)
    if "small" not in parts and "full" not in parts:
        return
    gen_dir = OUT / "generated"
    gen_dir.mkdir(exist_ok=True)
    for name, make in SMALL.items():
        text = make().to_text()
        (gen_dir / f"{name}.circuit.txt").write_text(text)
        rc = ref.parse(text)
        for level in (0, 1, 2):
            dem, _ = rc.compile(level)
            (gen_dir / f"{name}.L{level}.dem").write_text(dem)
        print(name, flush=True)
    full = {}
    for name, (make, levels) in FULL.items():
        text = make().to_text()
        rc = ref.parse(text)
        entry = {"circuit_sha256": sha(text), "levels": {}}
        for level in levels:
            t0 = time.time()
            dem, st = rc.compile(level)
            entry["levels"][str(level)] = {"edges": st["edges"], "dem_sha256": sha(dem)}
            print(name, level, st["edges"], f"{time.time() - t0:.1f}s", flush=True)
        full[name] = entry
    branches = []
    for b in range(BRANCHES):
        text = gp.gen_bb72_branch(b).to_text()
        dem, st = ref.parse(text).compile(0)
        branches.append({"branch": b, "circuit_sha256": sha(text), "edges": st["edges"], "dem_sha256": sha(dem)})
    full["bb72_branches_r6_L0"] = {"seed": 1, "branches": branches}
    (OUT / "full_size.json").write_text(json.dumps(full, indent=1) + "\n")


if __name__ == "__main__":
    main()

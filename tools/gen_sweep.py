"""Device-generated branch batches: wall time per call under GP_GEN_SUB
variants (developer tool)."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_16613_b200 as gp  # noqa: E402

spec = gp.bb72_branch_spec()
for v in sys.argv[1:]:
    os.environ["GP_GEN_SUB"] = v
    comp = gp.Compiler(0)
    for _ in range(3):
        comp.compile_bb_branches_raw(spec, 0, 4096, 0)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        comp.compile_bb_branches_raw(spec, 0, 4096, 0)
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"GP_GEN_SUB={v}: median {ts[5] * 1e3:.2f} ms  min {ts[0] * 1e3:.2f}", flush=True)

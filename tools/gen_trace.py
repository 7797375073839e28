"""Pipeline trace of device-generated vs host-circuit branch batches
(GP_PIPE_TRACE=1 prints per sub-batch host / device times; developer tool)."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2604_16613_b200 as gp  # noqa: E402

comp = gp.Compiler(0)
spec = gp.bb72_branch_spec()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
for i in range(4):
    t0 = time.perf_counter()
    out, st = comp.compile_bb_branches_raw(spec, 0, n, 0)
    print(f"gen call {i}: {(time.perf_counter() - t0) * 1e3:.2f} ms  kernel {st['kernel_ns'] / 1e6:.2f} "
          f"lower {st['lower_ns'] / 1e6:.2f}", file=sys.stderr, flush=True)
circuits = bench.build_branches(0, n)  # (the views point into these)
views = bench.views_of(circuits)
for i in range(4):
    t0 = time.perf_counter()
    out, st = comp.compile_batch_raw(views, 0)
    print(f"host call {i}: {(time.perf_counter() - t0) * 1e3:.2f} ms", file=sys.stderr, flush=True)

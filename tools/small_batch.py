"""Latency of gp_compile_batch for small batches of BB72 r6 branches (developer
tool: what a combined batch of concurrent drop-in calls costs)."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2604_16613_b200 as gp  # noqa: E402

comp = gp.Compiler(0)
for n in (1, 4, 8, 16, 64):
    gens = [gp.gen_bb72_branch(b) for b in range(n)]
    views = bench.views_of(gens)
    ts, ks = [], []
    for i in range(200):
        out, st = comp.compile_batch_raw(views, 0)
        if i >= 20:
            ts.append(st["total_ns"] / 1e3)
            ks.append(st["kernel_ns"] / 1e3)
    print(f"batch {n:3d}: total p50 {statistics.median(ts):7.1f} us  kernels {statistics.median(ks):7.1f} us  "
          f"launches {st['kernel_launches']}", flush=True)

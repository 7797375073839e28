"""Stage times of the 4,096-branch bench workload under environment variants
(developer tool; tuning knobs are read by the library at plan time).
usage: python tools/stage_sweep.py 'GP_TRAV_WARPS=2,4' 'GP_TRAV_WARPS=2,6;GP_X=1' ...
Each variant: one compile (pipelining off), parity against the reference
digests, then 10 CUDA-event-timed replays with live per-stage times."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2604_16613_b200 as gp  # noqa: E402


class _D:
    def sum(self, x):
        return x


variants = sys.argv[1:] or [""]
circuits = bench.build_branches(0, 4096)
views = bench.views_of(circuits)
keys = set()
for v in variants:
    for kv in filter(None, v.split(";")):
        if not kv.startswith("OPT99"):
            keys.add(kv.split("=")[0])
for v in variants:
    for k in keys:
        os.environ.pop(k, None)
    opt99 = 0
    for kv in filter(None, v.split(";")):
        k, x = kv.split("=", 1)
        if k == "OPT99":  # traversal experiments (gp_set_option 99): parity not expected
            opt99 = int(x)
        else:
            os.environ[k] = x
    comp = gp.Compiler(0)
    comp.set_option(bench.OPT_PIPELINE, 0)
    if opt99:
        comp.set_option(99, opt99)
    for _ in range(2):
        out, st = comp.compile_batch_raw(views, 0)
    par = bench.branch_parity(comp, out, 0, 4096, _D())
    comp.replay(3, True)
    rep = comp.replay(10, True)
    prof = comp.profile_stages()
    stages = " ".join(f"{k}={v / 1e6:.3f}" for k, v in prof.items() if v > 20000)
    print(f"[{v or 'default'}] {rep['kernel_ns'] / 10 / 1e6:.3f} ms/step  mism={par['mismatches']}  {stages}", flush=True)
    del comp

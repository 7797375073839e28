"""End-to-end batch time (pipelined public API, host circuits and device
generation) under pipeline knob variants (developer tool):
  python tools/e2e_sweep.py 'GP_PIPE_LANES=4' 'GP_PIPE_RAMP=1;GP_PIPE_SUB=384' ..."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2604_16613_b200 as gp  # noqa: E402

circuits = bench.build_branches(0, 4096)
views = bench.views_of(circuits)
spec = gp.bb72_branch_spec()
keys = {kv.split("=")[0] for v in sys.argv[1:] for kv in filter(None, v.split(";"))}
for v in sys.argv[1:] or [""]:
    for k in keys:
        os.environ.pop(k, None)
    for kv in filter(None, v.split(";")):
        k, x = kv.split("=", 1)
        os.environ[k] = x
    comp = gp.Compiler(0)
    res = {}
    for name, call in (("host", lambda: comp.compile_batch_raw(views, 0)),
                       ("gen", lambda: comp.compile_bb_branches_raw(spec, 0, 4096, 0))):
        for _ in range(3):
            call()
        ts = []
        for _ in range(9):
            t0 = time.perf_counter()
            call()
            ts.append(time.perf_counter() - t0)
        ts.sort()
        res[name] = ts[4] * 1e3
    print(f"[{v or 'default'}] host {res['host']:.2f} ms  gen {res['gen']:.2f} ms", flush=True)
    del comp

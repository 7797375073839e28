"""Timeline of one pipelined 4,096-branch compile, from host circuits and
generated on the device (developer tool): GP_PIPE_TRACE=1 prints, per sub-batch, the host pack
interval and the upload / kernels / download intervals on the device (us
from the batch start). Knobs as for e2e_sweep.py: python tools/pipe_trace.py 'GP_PIPE_SUB=384' ..."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2604_16613_b200 as gp  # noqa: E402

circuits = bench.build_branches(0, 4096)
views = bench.views_of(circuits)
for v in sys.argv[1:] or [""]:
    for kv in filter(None, v.split(";")):
        k, x = kv.split("=", 1)
        os.environ[k] = x
    comp = gp.Compiler(0)
    spec = gp.bb72_branch_spec()
    for name, call in (("host", lambda: comp.compile_batch_raw(views, 0)),
                       ("gen", lambda: comp.compile_bb_branches_raw(spec, 0, 4096, 0))):
        for _ in range(4):
            call()
        print(f"--- [{v or 'default'}] {name} traced:", file=sys.stderr, flush=True)
        os.environ["GP_PIPE_TRACE"] = "1"
        t0 = time.perf_counter()
        call()
        print(f"[{v or 'default'}] {name} wall {1e3 * (time.perf_counter() - t0):.2f} ms", file=sys.stderr, flush=True)
        os.environ.pop("GP_PIPE_TRACE")
    del comp

"""Single-circuit compile p50 (developer tool): total and device time of
gp_compile over repeated compiles of the bench's single circuits."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_16613_b200 as gp  # noqa: E402

cases = {"d3_L0": (lambda: gp.gen_surface(3, 3, 1e-3), 0),
         "d11_si1000_L2": (lambda: gp.gen_surface(11, 11, 1e-3, gp.NOISE_MODEL_SI1000), 2),
         "bb144_L0": (lambda: gp.gen_bb144(), 0), "bb144_L2": (lambda: gp.gen_bb144(), 2),
         "d25_L0": (lambda: gp.gen_surface(25, 25, 1e-3), 0)}
comp = gp.Compiler(0)
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 300
for name, (mk, lvl) in cases.items():
    g = mk()
    for _ in range(30):
        comp.compile(g, lvl)
    tot, ker = [], []
    for _ in range(iters):
        comp.compile(g, lvl)
        tot.append(comp.last_stats["total_ns"])
        ker.append(comp.last_stats["kernel_ns"])
    tot.sort()
    ker.sort()
    print(f"{name:16s} p50 total {tot[iters // 2] / 1e3:8.1f} us  kernel {ker[iters // 2] / 1e3:8.1f} us", flush=True)

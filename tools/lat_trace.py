"""Host-phase breakdown of single small compiles (GP_LAT_TRACE=1; developer tool)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_16613_b200 as gp  # noqa: E402

g = gp.gen_surface(3, 3, 1e-3)
comp = gp.Compiler(0)
for _ in range(200):
    comp.compile(g, 0)
tot, ker = [], []
for _ in range(2000):
    comp.compile(g, 0)
    tot.append(comp.last_stats["total_ns"])
    ker.append(comp.last_stats["kernel_ns"])
tot.sort()
ker.sort()
print(f"p50 total {tot[1000] / 1e3:.1f} us  kernel {ker[1000] / 1e3:.1f} us", file=sys.stderr, flush=True)

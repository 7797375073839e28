"""Single small compiles (developer tool): p50 of gp_compile total and device
time over 2,000 compiles of surface d3 r3 L0; GP_LAT_TRACE=1 prints the host
phases of each call; --phases prints the one-CTA kernel's phase timestamps
(option 99 bit 2)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_16613_b200 as gp  # noqa: E402

g = gp.gen_surface(3, 3, 1e-3)
comp = gp.Compiler(0)
for _ in range(200):
    comp.compile(g, 0)
if "--phases" in sys.argv:
    comp.set_option(99, 4)
    for _ in range(5):
        comp.compile(g, 0)
    sys.exit(0)
tot, ker = [], []
for _ in range(2000):
    comp.compile(g, 0)
    tot.append(comp.last_stats["total_ns"])
    ker.append(comp.last_stats["kernel_ns"])
tot.sort()
ker.sort()
print(f"p50 total {tot[1000] / 1e3:.1f} us  kernel {ker[1000] / 1e3:.1f} us", file=sys.stderr, flush=True)

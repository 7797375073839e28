"""A few compiles of one small circuit (for ncu captures of the one-CTA path)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_16613_b200 as gp  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 0
g = gp.gen_surface(3, 3, 1e-3)
comp = gp.Compiler(0)
for _ in range(5):
    d = comp.compile(g, level)
print(d.num_edges, comp.last_stats)

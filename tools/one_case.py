"""Compile a single named case once (debugging under compute-sanitizer)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_16613_b200 as gp
name, lv = sys.argv[1], int(sys.argv[2])
g = {"bb144": lambda: gp.gen_bb144(), "surf5": lambda: gp.gen_surface(5, 3, 1e-3),
     "bb72": lambda: gp.gen_bb(6, 6, rounds=2)}[name]()
d = gp.Compiler(0).compile(g, lv)
print(name, lv, d.num_edges)

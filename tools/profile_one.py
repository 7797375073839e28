"""Compile one workload a few times (for ncu captures; `--workload d3` is the
one-CTA small path)."""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_16613_b200 as gp

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="bb144")
ap.add_argument("--level", type=int, default=2)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--branches", type=int, default=512)
a = ap.parse_args()
comp = gp.Compiler(0)
if a.workload == "branches":
    gens = [gp.gen_bb72_branch(b) for b in range(a.branches)]
    for _ in range(a.iters):
        comp.compile_batch(gens, a.level)
else:
    g = {"bb144": lambda: gp.gen_bb144(), "d11": lambda: gp.gen_surface(11, 11, 1e-3, gp.NOISE_MODEL_SI1000),
         "d25": lambda: gp.gen_surface(25, 25, 1e-3), "d3": lambda: gp.gen_surface(3, 3, 1e-3)}[a.workload]()
    for _ in range(a.iters):
        d = comp.compile(g, a.level)
    print(a.workload, d.num_edges, comp.last_stats)

"""Repro: same context, L0 then L2 on BB144."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_16613_b200 as gp
c = gp.Compiler(0)
g = gp.gen_bb144()
for lv in [int(x) for x in sys.argv[1:]]:
    d = c.compile(g, lv)
    print(lv, d.num_edges, flush=True)

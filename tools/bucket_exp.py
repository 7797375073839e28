"""Bucket-kernel experiments (developer tool): option 99 bits 256 (skip sort), 512 (skip groups)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_16613_b200 as gp
g = gp.gen_bb144()
for dbg in (0, 256, 512, 768):
    c = gp.Compiler(0)
    c.set_option(99, dbg)
    for _ in range(3):
        c.compile(g, 2)
    c.replay(10)
    st = c.profile_stages()
    print("debug", dbg, "bucket us", st["bucket"] / 10 / 1e3, flush=True)

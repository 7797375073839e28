"""Traversal role experiments: time with emission / node work disabled."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_16613_b200 as gp  # noqa: E402

g = gp.gen_bb144()
for lv in (0, 2):
    for dbg in (0, 1, 2, 3):
        c = gp.Compiler(0)
        c.set_option(99, dbg)
        ts = []
        for i in range(8):
            c.compile(g, lv)
            ts.append(c.last_stats["traverse_kernel_ns"])
        print("L%d debug=%d traverse_us=%.1f" % (lv, dbg, sorted(ts)[4] / 1e3), flush=True)

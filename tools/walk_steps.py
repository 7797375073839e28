"""Per-step walk timing (developer tool, option 99 bit 2): where each boundary's cycles go.
Row j: [0] group start (first step of a group only), [1] after the stage wait,
[2] after the node work, [3] after the per-boundary barrier."""
import os, sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_16613_b200 as gp
os.environ["GP_DEBUG_DUMP"] = "/tmp/walk_dbg.bin"
name = sys.argv[1] if len(sys.argv) > 1 else "bb144"
g = {"bb144": lambda: gp.gen_bb144(), "d11": lambda: gp.gen_surface(11, 11, 1e-3, 1),
     "d25": lambda: gp.gen_surface(25, 25, 1e-3)}[name]()
c = gp.Compiler(0)
for _ in range(3):
    c.compile(g, 0)
c.set_option(99, 4 | int(sys.argv[2]) if len(sys.argv) > 2 else 4)
c.compile(g, 0)
a = np.fromfile("/tmp/walk_dbg.bin", dtype=np.uint64).reshape(-1, 512, 4).astype(np.int64)
steps = (a[:, :, 3] != 0).sum(1)
cta = int(np.argmax(steps))
x = a[cta, :steps[cta]]
end = x[:, 3]
tot = np.diff(end)
comp = x[1:, 2] - np.maximum(x[1:, 1], end[:-1])
bar = x[1:, 3] - x[1:, 2]
waits = [(i, x[i, 1] - x[i, 0]) for i in range(len(x)) if x[i, 0]]
print(name, "ctas", len(steps), "max steps", steps[cta], "total cycles", end[-1] - x[0, 0] if x[0, 0] else end[-1] - x[0, 1])
print("per step cycles: median total %d compute %d barrier %d" % (np.median(tot), np.median(comp), np.median(bar)))
print("group waits (step, cycles):", waits[:12])

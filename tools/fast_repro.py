"""One batch compile of BB72 branch circuits (for ncu captures of the reduce)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_16613_b200 as gp  # noqa: E402
from bench import views_of  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
level = int(sys.argv[2]) if len(sys.argv) > 2 else 0
gens = [gp.gen_bb72_branch(b) for b in range(n)]
views = views_of(gens)
comp = gp.Compiler(0)
comp.set_option(4, 0)
for i in range(2):
    out, st = comp.compile_batch_raw(views, level)
    print(i, out.num_edges, st["kernel_ns"] / 1e6, flush=True)

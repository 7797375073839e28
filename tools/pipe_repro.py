"""Pipelined batch repro (developer tool): usage pipe_repro.py N ROUNDS; GP_PIPE_TRACE=1 prints per
sub-batch host pack time and device event times."""
import sys; sys.path.insert(0, '/root/repo')
import paper_2604_16613_b200 as gp
n = int(sys.argv[1]); r = int(sys.argv[2])
gens = [gp.gen_bb72_branch(b, rounds=r) for b in range(n)]
views = None
comp = gp.Compiler(0)
from bench import views_of
views = views_of(gens)
comp.set_option(4, -1)
for i in range(3):
    out, st = comp.compile_batch_raw(views, 0)
    print(i, out.num_edges, flush=True)

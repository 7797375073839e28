import sys, statistics
sys.path.insert(0, '/root/repo')
import paper_2604_16613_b200 as gp
c = gp.Compiler(0)
g = gp.gen_bb72_branch(7)
ks, ts, ls = [], [], []
for i in range(300):
    d = c.compile(g, 0)
    if i >= 50:
        ks.append(c.last_stats["kernel_ns"]); ts.append(c.last_stats["total_ns"]); ls.append(c.last_stats["kernel_launches"])
print("edges", d.num_edges, "kernel p50 us", statistics.median(ks)/1e3, "total p50 us", statistics.median(ts)/1e3, "launches", ls[-1])

"""Group-size and records-per-source histograms of a BB72 branch circuit (developer tool, GPU)."""
import sys; sys.path.insert(0,'/root/repo')
import numpy as np, collections
import paper_2604_16613_b200 as gp
comp = gp.Compiler(0)
for lv in (0,2):
    t = comp.compile_shard(gp.gen_bb72_branch(3), 0, 1, lv)
    sig = collections.Counter()
    for i in range(t.num_sources):
        a, b = t.rec_offsets[i], t.rec_offsets[i+1]
        key = tuple(sorted(zip(t.rec_words[a:b].tolist(), t.rec_bits[a:b].tolist())))
        sig[key] += 1
    sizes = np.array(list(sig.values()))
    print(lv, "sources", t.num_sources, "groups", len(sizes), "max", sizes.max(), "hist", np.histogram(sizes, bins=[1,2,3,5,9,17,33,65,129,10**6])[0].tolist())
    nrec = np.diff(t.rec_offsets)
    print("  records per source hist", np.bincount(nrec).tolist())

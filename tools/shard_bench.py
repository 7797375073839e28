"""Fault-range sharding timing on one GPU: each shard of a
single circuit compiled in turn (what rank k would run), the merge of all
partial tables, and the whole-circuit compile for comparison. Wall-clock per
call through the C ABI, p50 over repeats (host packing + upload included).
shard_ms keeps each partial table on the device (what a rank of
compile_sharded runs before the owner exchange); shard_host_table_ms also
copies it out to host arrays."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2604_16613_b200 as gp  # noqa: E402


def p50(f, reps):
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        r = f()
        ts.append(time.perf_counter() - t)
    return float(np.median(ts)) * 1e3, r


def main():
    comp = gp.Compiler(0)
    cases = {"surface_d25_r25": lambda: gp.gen_surface(25, 25, 1e-3),
             "bb144_r12": lambda: gp.gen_bb144(12, 1e-3)}
    out = {}
    for name, mk in cases.items():
        g = mk()
        for level in (0, 2):
            comp.compile(g, level)
            whole_ms, dem = p50(lambda: comp.compile(g, level), 7)
            want = dem.to_text()
            row = {"whole_ms": whole_ms, "edges": dem.num_edges}
            for n in (2, 4, 8):
                shard_ms, shard_host_ms, parts = [], [], []
                for k in range(n):
                    # a rank's shard as compile_sharded runs it: the partial
                    # table stays on the device for the owner exchange
                    comp.compile_shard(g, k, n, level, on_device=True)
                    ms, _ = p50(lambda: comp.compile_shard(g, k, n, level, on_device=True), 5)
                    shard_ms.append(ms)
                    # the same with the table copied out to host arrays
                    comp.compile_shard(g, k, n, level)
                    ms, part = p50(lambda: comp.compile_shard(g, k, n, level), 5)
                    shard_host_ms.append(ms)
                    parts.append(part)
                merge_ms, m = p50(lambda: comp.merge_partials(parts), 5)
                assert m.to_text() == want
                dparts = []
                for k in range(n):
                    t = comp.compile_shard(g, k, n, level, on_device=True)
                    dparts.append(gp.DevicePartialTable(t.num_detectors, t.num_observables,
                                                        *(x.clone() for x in t.arrays().values())))
                dmerge_ms, m = p50(lambda: comp.merge_partials(dparts), 5)
                assert m.to_text() == want
                dev_stats = comp.last_stats
                # the fold spread over owners (shard.compile_sharded): every
                # shard's entries split by owning rank; owner o merges its
                # pieces of all shards -- the per-rank merge time at n ranks
                # is the max over owners (each would run on its own GPU)
                from paper_2604_16613_b200 import shard
                pieces = []
                for k in range(n):
                    t = comp.compile_shard(g, k, n, level, on_device=True)
                    pieces.append(shard.split_by_owner(t.num_detectors, *(x.clone() for x in t.arrays().values()), n))
                owner_ms, owner_entries, texts = [], [], []
                for o in range(n):
                    mine = [gp.DevicePartialTable(parts[0].num_detectors, parts[0].num_observables, *pc[o])
                            for pc in pieces if pc[o][0].numel()]
                    ms_o, d_o = p50(lambda: comp.merge_partials(mine), 5)
                    owner_ms.append(ms_o)
                    owner_entries.append(int(sum(x.probs.numel() for x in mine)))
                    texts.append(d_o)
                assert shard.concat_dems(texts).to_text() == want
                nbytes = sum(p.probs.nbytes + p.rec_offsets.nbytes + p.rec_words.nbytes + p.rec_bits.nbytes
                             for p in parts)
                row[f"n{n}"] = {"shard_ms": [round(x, 3) for x in shard_ms], "max_shard_ms": max(shard_ms),
                                "shard_host_table_ms": [round(x, 3) for x in shard_host_ms],
                                "merge_ms": merge_ms, "merge_dev_ms": dmerge_ms,
                                "merge_dev_kernel_ms": dev_stats["kernel_ns"] / 1e6, "table_bytes": nbytes,
                                "owner_merge_ms": [round(x, 3) for x in owner_ms],
                                "max_owner_merge_ms": max(owner_ms), "owner_entries": owner_entries,
                                "sources": [p.num_sources for p in parts]}
            out[f"{name}_L{level}"] = row
            print(name, level, json.dumps(row), flush=True)
    json.dump(out, open("gpurun_out/shard_bench.json", "w"), indent=1)


if __name__ == "__main__":
    main()

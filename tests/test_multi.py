"""CPU, world_size 2 over gloo: the multi-GPU host logic of bench.py --
branch sharding (disjoint, weak scaling), max-over-ranks timing, summed
metric, and the final variable-size gather of per-rank DEM tables."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from .conftest import ROOT


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, str(ROOT))
    import bench
    import paper_2604_16613_b200 as gp
    try:
        dist = bench.Dist(world, "gloo")
        ids = list(bench.shard(rank, world, 3))
        circuits = [gp.gen_bb72_branch(b, rounds=3) for b in ids]
        # host-only stand-in for the per-rank DEM table: detector counts
        nd = np.array([c.num_detectors for c in circuits], np.uint32)
        total = dist.sum(float(nd.sum()))
        tmax = dist.max(float(rank + 1))
        got = bench.gather_flat(dist, {"ids": np.array(ids, np.uint32), "nd": nd,
                                       "p": np.arange(len(ids) + rank, dtype=np.float64)}, "cpu")
        dist.close()
        q.put((rank, ids, float(nd.sum()), total, tmax, {k: [x.tolist() for x in v] for k, v in got.items()}))
    except Exception as e:  # pragma: no cover
        q.put((rank, "error", repr(e)))


def test_two_rank_sharding_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    [p.start() for p in procs]
    res = sorted([q.get(timeout=120) for _ in procs])
    [p.join(timeout=60) for p in procs]
    for r in res:
        assert r[1] != "error", r
    (r0, ids0, s0, tot0, max0, g0), (r1, ids1, s1, tot1, max1, g1) = res
    assert not set(ids0) & set(ids1) and sorted(ids0 + ids1) == list(range(6))
    assert tot0 == tot1 == s0 + s1
    assert max0 == max1 == 2.0
    assert g0 == g1
    assert g0["ids"] == [ids0, ids1]
    assert [len(x) for x in g0["p"]] == [3, 4]  # ragged per-rank tables

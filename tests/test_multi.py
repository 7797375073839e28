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


def _shard_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, str(ROOT))
    import torch.distributed as td
    from paper_2604_16613_b200 import shard
    from paper_2604_16613_b200.api import PartialTable
    try:
        td.init_process_group("gloo")
        rng = np.random.default_rng(rank)
        n = 3 + 4 * rank  # ragged per-rank tables
        cnt = rng.integers(1, 4, n)
        roff = np.concatenate([[0], np.cumsum(cnt)]).astype(np.uint32)
        r = int(roff[-1])
        t = PartialTable(100, 2, rng.random(n), roff, rng.integers(0, 2, r).astype(np.uint32),
                         rng.integers(0, 2**64, r, dtype=np.uint64) | np.uint64(1 << 63))
        got = shard.tables_from(shard.gather_flat(shard.table_arrays(t), "cpu"))
        td.destroy_process_group()
        q.put((rank, [(g.num_detectors, g.num_observables, g.probs.tobytes(), g.rec_offsets.tobytes(),
                       g.rec_words.tobytes(), g.rec_bits.tobytes()) for g in got],
               (t.probs.tobytes(), roff.tobytes(), t.rec_words.tobytes(), t.rec_bits.tobytes())))
    except Exception as e:  # pragma: no cover
        q.put((rank, "error", repr(e)))


def test_two_rank_partial_table_gather_is_bit_exact():
    """The fault-range sharding exchange (paper_2604_16613_b200.shard): ragged
    partial tables (f64 probabilities, u64 records with the top bit set)
    reach every rank bit-exactly, in rank order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    [p.start() for p in procs]
    res = sorted([q.get(timeout=120) for _ in procs], key=lambda x: x[0])
    [p.join(timeout=60) for p in procs]
    for r in res:
        assert r[1] != "error", r
    own = [r[2] for r in res]
    for _, got, _ in res:
        assert [g[:2] for g in got] == [(100, 2), (100, 2)]
        assert [g[2:] for g in got] == own


def test_shard_layer_ranges_partition():
    from paper_2604_16613_b200.shard import shard_of
    for layers in (1, 5, 17, 100):
        for world in (1, 2, 3, 8, 13):
            rs = [shard_of(k, world, layers) for k in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == layers
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))

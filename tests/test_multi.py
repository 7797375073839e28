"""CPU, world_size 2 over gloo: the multi-GPU host logic -- branch sharding
(disjoint, weak scaling), max-over-ranks timing, summed metric, the final
variable-size gather of per-rank DEM tables to rank 0, and the fault-range
sharding exchange (paper_2604_16613_b200.shard): ownership of signatures by
canonical range, the all-to-all of partial-table entries to their owners,
the owners' DEMs concatenated in canonical order. (The same paths with real
GPU compiles: tests/test_gpu.py::test_two_process_*.)"""

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
        q.put((rank, ids, float(nd.sum()), total, tmax,
               None if got is None else {k: [x.tolist() for x in v] for k, v in got.items()}))
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
    assert g1 is None  # gathered to rank 0 only
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


def _synthetic_table(rng, D, O, n):
    """A partial table with known first detectors: entry i's records are
    distinct words with random bits, its first detector recorded."""
    from paper_2604_16613_b200.api import PartialTable
    W = (D + O + 63) // 64
    probs, offs, words, bits, first = [], [0], [], [], []
    for _ in range(n):
        k = int(rng.integers(1, min(W, 4) + 1))
        ws = sorted(rng.choice(W, size=k, replace=False).tolist())
        ids = set()
        for w in ws:
            b = int(rng.integers(1, 2**63)) | (1 << int(rng.integers(0, 64)))
            lim = min(64, D + O - 64 * w)
            b &= (1 << lim) - 1 if lim < 64 else (1 << 64) - 1
            if b == 0:
                b = 1
            words.append(w)
            bits.append(b)
            ids |= {64 * w + x for x in range(64) if b >> x & 1}
        dets = [x for x in ids if x < D]
        first.append(min(dets) if dets else -1)
        probs.append(float(rng.random()))
        offs.append(len(words))
    t = PartialTable(D, O, np.array(probs), np.array(offs, np.uint32), np.array(words, np.uint32),
                     np.array(bits, np.uint64))
    return t, np.array(first)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_owner_partition(world):
    """entry_owners: an entry goes to the rank whose canonical range holds its
    first detector + 1 (0 for observable-only); split_by_owner keeps every
    entry exactly once with its records, in table order."""
    import torch

    from paper_2604_16613_b200 import shard
    rng = np.random.default_rng(world)
    D, O = 300, 70
    t, first = _synthetic_table(rng, D, O, 400)
    w = shard.table_arrays(t)
    tab = tuple(shard._to_wire(w[k]) for k in ("probs", "rec_offsets", "rec_words", "rec_bits"))
    own = shard.entry_owners(D, *tab, world).numpy()
    b = shard.owner_bounds(D, world)
    q0 = first + 1
    assert all(b[o] <= q <= b[o + 1] - 1 for o, q in zip(own, q0))
    pieces = shard.split_by_owner(D, *tab, world)
    assert sum(p[0].numel() for p in pieces) == 400
    for r, (pr, off, wd, bt) in enumerate(pieces):
        idx = np.nonzero(own == r)[0]
        assert np.array_equal(pr.numpy(), t.probs[idx])
        recs = [(int(t.rec_words[j]), int(t.rec_bits[j])) for i in idx
                for j in range(t.rec_offsets[i], t.rec_offsets[i + 1])]
        assert list(zip(wd.numpy().view(np.uint32).tolist(), bt.numpy().view(np.uint64).tolist())) == recs
        assert off.numpy()[-1] == len(recs)


def test_concat_dems_rebases_offsets():
    from paper_2604_16613_b200 import shard
    from paper_2604_16613_b200.api import Dem
    a = Dem(5, 1, np.array([0, 2, 3], np.uint32), np.array([0, 1, 4], np.uint32), np.array([0, 0, 1], np.uint32),
            np.array([0], np.uint32), np.array([0.1, 0.2]))
    e = Dem(5, 1, np.array([0], np.uint32), np.zeros(0, np.uint32), np.array([0], np.uint32), np.zeros(0, np.uint32),
            np.zeros(0))
    b = Dem(5, 1, np.array([0, 1], np.uint32), np.array([3], np.uint32), np.array([0, 1], np.uint32),
            np.array([0], np.uint32), np.array([0.3]))
    c = shard.concat_dems([a, e, b])
    assert c.hyperedges() == a.hyperedges() + b.hyperedges()


def _exchange_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, str(ROOT))
    import torch.distributed as td

    from paper_2604_16613_b200 import shard
    try:
        td.init_process_group("gloo")
        rng = np.random.default_rng(10 + rank)
        D, O = 200, 12
        t, first = _synthetic_table(rng, D, O, 50 + 30 * rank)
        w = shard.table_arrays(t)
        tab = tuple(shard._to_wire(w[k]) for k in ("probs", "rec_offsets", "rec_words", "rec_bits"))
        got = shard.exchange_by_owner(shard.split_by_owner(D, *tab, world))
        td.destroy_process_group()
        q.put((rank, [tuple(x.numpy().tobytes() for x in p) for p in got],
               [tuple(x.numpy().tobytes() for x in p) for p in shard.split_by_owner(D, *tab, world)]))
    except Exception as e:  # pragma: no cover
        q.put((rank, "error", repr(e)))


def test_two_rank_owner_exchange():
    """All-to-all of partial-table pieces by owner over gloo: rank r receives,
    from each rank s in order, exactly the piece s cut for r (bit-exact)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    [p.start() for p in procs]
    res = sorted([q.get(timeout=120) for _ in procs], key=lambda x: x[0])
    [p.join(timeout=60) for p in procs]
    for r in res:
        assert r[1] != "error", r
    cut = {r: res[r][2] for r in range(2)}  # cut[s][r]: the piece rank s made for r
    for r in range(2):
        assert res[r][1] == [cut[s][r] for s in range(2)]

"""Multi-GPU compile of ONE circuit by fault-range sharding,
and the final gather of per-rank DEM tables.

Rank k of n runs gp_compile_shard on its GPU: the walk (Alg. 1, stepg.cpp)
of every detector word down to the shard's first layer only, and the
emission of the error sources placed in layers [l*k/n, l*(k+1)/n) -- their
noise ops and the outcome flips of their measurements. The result is a
partial table of UNFOLDED signatures (one entry per nonempty source), so the
exchange ships constituent probabilities and every fold is bit-exact
(dem.cpp:97-106 folds a group's sorted member probabilities).

The fold is spread over the ranks: every entry is
sent to the rank that OWNS its signature (all-to-all of the partial tables,
grouped point-to-point sends / receives: ncclGroupStart / ncclSend /
ncclRecv over NVLink under NCCL), each owner merges what it received
(gp_merge_partials: bucket / group / fold / write on its device) and the
owners' DEMs are gathered to the root. Ownership is a RANGE of the canonical
order, not a hash: rank r owns the signatures whose first detector + 1 (0 for
observable-only signatures, which sort first, dem.cpp:122-127) lies in
[r (D + 1) / n, (r + 1) (D + 1) / n). Identical signatures share their first
detector, so all members of a group meet at one owner, and the owners' DEMs
concatenated in rank order are already in canonical order -- the root only
rebases offsets. The reference has no multi-GPU path; the
result equals demc::compile_circuit (compile.cpp:23-53) of the whole circuit.

Arrays travel bit-exactly: u32 as int32, u64 as int64 views, f64 as is.
"""

from __future__ import annotations

import numpy as np

from .api import CorrelationLevel, Dem, PartialTable  # noqa: F401

_WIRE = {np.dtype(np.uint32): np.int32, np.dtype(np.uint64): np.int64, np.dtype(np.int32): np.int32,
         np.dtype(np.int64): np.int64, np.dtype(np.float64): np.float64}
_UNWIRE = {np.dtype(np.int32): np.uint32, np.dtype(np.int64): np.uint64, np.dtype(np.float64): np.float64}


def _to_wire(a: np.ndarray):
    import torch
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a.view(_WIRE[a.dtype]).copy())


def gather_flat(arrays: dict, device: str, group=None) -> dict:
    """All-gathers variable-length flat arrays: per array one all_gather of
    the lengths, then one of the payloads padded to the longest. Returns
    {name: [per-rank np.ndarray]} on every rank, dtypes preserved bit-exactly.
    (Kept for callers that need the tables everywhere; the DEM exchange uses
    gather_to_root.)"""
    import torch
    import torch.distributed as td

    ws = td.get_world_size(group)
    out = {}
    for name, a in arrays.items():
        a = np.ascontiguousarray(a)
        t = _to_wire(a).to(device)
        n = torch.tensor([t.numel()], dtype=torch.int64, device=device)
        sizes = [torch.zeros_like(n) for _ in range(ws)]
        td.all_gather(sizes, n, group=group)
        lens = [int(x.item()) for x in sizes]
        pad = torch.zeros(max(max(lens), 1), dtype=t.dtype, device=device)
        pad[:t.numel()] = t
        parts = [torch.zeros_like(pad) for _ in range(ws)]
        td.all_gather(parts, pad, group=group)
        out[name] = [parts[r][:lens[r]].cpu().numpy().view(a.dtype) for r in range(ws)]
    return out


def _lengths(tensors: list, device, group) -> list[list[int]]:
    """[rank][i] = numel of tensor i on each rank (one all_gather)."""
    import torch
    import torch.distributed as td

    ws = td.get_world_size(group)
    mine = torch.tensor([t.numel() for t in tensors], dtype=torch.int64, device=device)
    got = [torch.zeros_like(mine) for _ in range(ws)]
    td.all_gather(got, mine, group=group)
    return [[int(x) for x in g.tolist()] for g in got]


def _p2p(ops: list) -> None:
    """Grouped point-to-point (NCCL: one ncclGroupStart/End around the sends
    and receives)."""
    import torch.distributed as td
    if ops:
        for req in td.batch_isend_irecv(ops):
            req.wait()


def gather_tensors_to_root(tensors: dict, root: int = 0, group=None) -> dict | None:
    """Variable-size gather of flat tensors to `root` (exact-size buffers;
    grouped sends / receives, no padding, no copy on the other ranks).
    Returns {name: [per-rank tensor]} on root, None elsewhere."""
    import torch
    import torch.distributed as td

    rank, ws = td.get_rank(group), td.get_world_size(group)
    names = list(tensors)
    ts = [tensors[k].contiguous() for k in names]
    dev = ts[0].device if ts else torch.device("cpu")
    lens = _lengths(ts, dev, group)
    groot = td.get_global_rank(group, root) if group is not None else root
    if rank != root:
        _p2p([td.P2POp(td.isend, t, groot, group) for t in ts if t.numel()])
        return None
    out = {k: [None] * ws for k in names}
    ops = []
    for r in range(ws):
        for i, k in enumerate(names):
            if r == root:
                out[k][r] = ts[i]
                continue
            buf = torch.empty(lens[r][i], dtype=ts[i].dtype, device=dev)
            out[k][r] = buf
            if buf.numel():
                src = td.get_global_rank(group, r) if group is not None else r
                ops.append(td.P2POp(td.irecv, buf, src, group))
    _p2p(ops)
    return out


def gather_to_root(arrays: dict, device: str, root: int = 0, group=None) -> dict | None:
    """gather_tensors_to_root for numpy arrays (through `device`: "cpu" for
    gloo, "cuda:k" for NCCL). {name: [per-rank np.ndarray]} on root."""
    dtypes = {k: np.ascontiguousarray(a).dtype for k, a in arrays.items()}
    got = gather_tensors_to_root({k: _to_wire(a).to(device) for k, a in arrays.items()}, root, group)
    if got is None:
        return None
    return {k: [t.cpu().numpy().view(dtypes[k]) for t in v] for k, v in got.items()}


def table_arrays(t: PartialTable) -> dict:
    """The wire form of a partial table (shapes recorded in `dims`)."""
    return {"dims": np.array([t.num_detectors, t.num_observables], np.int64),
            "probs": np.ascontiguousarray(t.probs, np.float64),
            "rec_offsets": np.ascontiguousarray(t.rec_offsets, np.uint32),
            "rec_words": np.ascontiguousarray(t.rec_words, np.uint32),
            "rec_bits": np.ascontiguousarray(t.rec_bits, np.uint64)}


def tables_from(gathered: dict) -> list[PartialTable]:
    out = []
    for r in range(len(gathered["dims"])):
        d = gathered["dims"][r]
        out.append(PartialTable(int(d[0]), int(d[1]), gathered["probs"][r], gathered["rec_offsets"][r],
                                gathered["rec_words"][r], gathered["rec_bits"][r]))
    return out


def shard_of(rank: int, world: int, num_layers: int) -> tuple[int, int]:
    """Layer range [lo, hi) of shard `rank` (the split gp_compile_shard uses)."""
    return num_layers * rank // world, num_layers * (rank + 1) // world


def owner_bounds(num_detectors: int, world: int) -> list[int]:
    """Rank r owns canonical buckets q0 in [b[r], b[r + 1]) (q0 = first
    detector + 1; 0 = no detector)."""
    return [(num_detectors + 1) * r // world for r in range(world + 1)]


def entry_owners(num_detectors: int, probs, rec_offsets, rec_words, rec_bits, world: int):
    """Owner rank of every entry of a partial table (torch tensors on any
    device: int32 offsets / words, int64 bits = the u32 / u64 bit patterns).
    The first detector of an entry is the lowest detector bit of its records
    (records carry distinct words; a word's bits below D are detectors)."""
    import torch

    dev = rec_bits.device
    n = probs.numel()
    if n == 0:
        return torch.zeros(0, dtype=torch.int64, device=dev)
    D = int(num_detectors)
    w = rec_words.to(torch.int64)
    base = w * 64
    span = (D - base).clamp(0, 64)  # detector bits of each record's word
    mask = torch.where(span >= 64, torch.full_like(base, -1),
                       torch.bitwise_left_shift(torch.ones_like(base), span.clamp(max=63)) - 1)
    det = rec_bits & mask
    low = det & (-det)  # isolated lowest set bit (two's complement; bit 63 -> INT64_MIN)
    bit = torch.where(low < 0, torch.full_like(low, 63), torch.log2(low.to(torch.float64).abs()).to(torch.int64))
    big = torch.full_like(base, 1 << 40)
    first = torch.where(det != 0, base + bit, big)
    cnt = (rec_offsets[1:] - rec_offsets[:-1]).to(torch.int64)
    ent = torch.repeat_interleave(torch.arange(n, device=dev), cnt)
    fmin = torch.full((n,), 1 << 40, dtype=torch.int64, device=dev).scatter_reduce(0, ent, first, reduce="amin")
    q0 = torch.where(fmin >= (1 << 40), torch.zeros_like(fmin), fmin + 1)
    b = torch.tensor(owner_bounds(D, world), dtype=torch.int64, device=dev)
    return torch.searchsorted(b, q0, right=True) - 1


def split_by_owner(num_detectors: int, probs, rec_offsets, rec_words, rec_bits, world: int) -> list[tuple]:
    """Per owner rank: (probs, rec_offsets, rec_words, rec_bits) of the
    entries it owns, in table order (torch tensors, wire dtypes)."""
    import torch

    own = entry_owners(num_detectors, probs, rec_offsets, rec_words, rec_bits, world)
    cnt = (rec_offsets[1:] - rec_offsets[:-1]).to(torch.int64)
    rec_own = torch.repeat_interleave(own, cnt)
    out = []
    for r in range(world):
        sel = own == r
        rsel = rec_own == r
        c = cnt[sel]
        off = torch.zeros(c.numel() + 1, dtype=torch.int64, device=probs.device)
        off[1:] = torch.cumsum(c, 0)
        out.append((probs[sel].contiguous(), off.to(torch.int32), rec_words[rsel].contiguous(),
                    rec_bits[rsel].contiguous()))
    return out


def exchange_by_owner(parts: list[tuple], group=None) -> list[tuple]:
    """All-to-all of per-owner table pieces: parts[r] goes to rank r; returns
    the pieces every rank sent to this one, in source-rank order (grouped
    sends / receives; NCCL: one ncclGroupStart/End)."""
    import torch
    import torch.distributed as td

    rank, ws = td.get_rank(group), td.get_world_size(group)
    flat = [t for p in parts for t in p]
    dev = flat[0].device
    lens = _lengths(flat, dev, group)  # [src][4 * dst + i]
    recv = [[None] * 4 for _ in range(ws)]
    ops = []
    for r in range(ws):
        for i in range(4):
            if r == rank:
                recv[r][i] = parts[rank][i]
                continue
            buf = torch.empty(lens[r][4 * rank + i], dtype=parts[rank][i].dtype, device=dev)
            recv[r][i] = buf
            peer = td.get_global_rank(group, r) if group is not None else r
            if buf.numel():
                ops.append(td.P2POp(td.irecv, buf, peer, group))
            if parts[r][i].numel():
                ops.append(td.P2POp(td.isend, parts[r][i].contiguous(), peer, group))
    _p2p(ops)
    return [tuple(x) for x in recv]


def concat_dems(dems: list[Dem]) -> Dem:
    """Owners' DEMs in rank order -> one DEM (offsets rebased)."""
    d0 = dems[0]
    det_off, obs_off = [np.zeros(1, np.uint32)], [np.zeros(1, np.uint32)]
    nd = no = 0
    for d in dems:
        det_off.append((np.asarray(d.det_offsets[1:], np.uint64) + nd).astype(np.uint32))
        obs_off.append((np.asarray(d.obs_offsets[1:], np.uint64) + no).astype(np.uint32))
        nd += int(d.det_offsets[-1]) if len(d.det_offsets) else 0
        no += int(d.obs_offsets[-1]) if len(d.obs_offsets) else 0
    return Dem(d0.num_detectors, d0.num_observables, np.concatenate(det_off),
               np.concatenate([np.asarray(d.det_ids, np.uint32) for d in dems]), np.concatenate(obs_off),
               np.concatenate([np.asarray(d.obs_ids, np.uint32) for d in dems]),
               np.concatenate([np.asarray(d.probs, np.float64) for d in dems]))


def _dem_arrays(d: Dem) -> dict:
    return {"det_offsets": np.asarray(d.det_offsets, np.uint32), "det_ids": np.asarray(d.det_ids, np.uint32),
            "obs_offsets": np.asarray(d.obs_offsets, np.uint32), "obs_ids": np.asarray(d.obs_ids, np.uint32),
            "probs": np.asarray(d.probs, np.float64)}


def compile_sharded(compiler, circuit, level=CorrelationLevel.L0, group=None, root: int | None = 0,
                    timings: dict | None = None) -> Dem | None:
    """One circuit compiled across the ranks of `group` (torch.distributed
    initialised; one process per GPU, compiler on that GPU): shard compile ->
    all-to-all of the partial tables by owner -> each owner merges (folds)
    its signatures -> the owners' DEMs gathered to `root` (every rank when
    root is None). Over NCCL the tables stay in HBM (compile_shard(on_device
    =True), NVLink point-to-point, merge from device memory); over gloo they
    go through the host. `timings` (optional) receives per-phase seconds."""
    import time

    import torch
    import torch.distributed as td

    from .api import DevicePartialTable

    rank, world = td.get_rank(group), td.get_world_size(group)
    nccl = td.get_backend(group) == "nccl"
    t0 = time.perf_counter()
    if nccl:
        part = compiler.compile_shard(circuit, rank, world, level, on_device=True)
        a = part.arrays()
        tab = (a["probs"], a["rec_offsets"], a["rec_words"], a["rec_bits"])
    else:
        part = compiler.compile_shard(circuit, rank, world, level)
        w = table_arrays(part)
        tab = tuple(_to_wire(w[k]) for k in ("probs", "rec_offsets", "rec_words", "rec_bits"))
    D, O = part.num_detectors, part.num_observables
    t1 = time.perf_counter()
    mine = exchange_by_owner(split_by_owner(D, *tab, world), group)
    t2 = time.perf_counter()
    if nccl:
        parts = [DevicePartialTable(D, O, *p) for p in mine if p[0].numel()]
    else:
        parts = [PartialTable(D, O, p[0].numpy(), p[1].numpy().view(np.uint32), p[2].numpy().view(np.uint32),
                              p[3].numpy().view(np.uint64)) for p in mine if p[0].numel()]
    if parts:
        dem = compiler.merge_partials(parts)
    else:
        dem = Dem(D, O, np.zeros(1, np.uint32), np.zeros(0, np.uint32), np.zeros(1, np.uint32),
                  np.zeros(0, np.uint32), np.zeros(0, np.float64))
    t3 = time.perf_counter()
    dev = f"cuda:{torch.cuda.current_device()}" if nccl else "cpu"
    out = None
    if root is None:
        got = gather_flat(_dem_arrays(dem), dev, group)
        out = concat_dems([Dem(D, O, *(got[k][r] for k in ("det_offsets", "det_ids", "obs_offsets", "obs_ids",
                                                               "probs"))) for r in range(world)])
    else:
        got = gather_to_root(_dem_arrays(dem), dev, root, group)
        if got is not None:
            out = concat_dems([Dem(D, O, *(got[k][r] for k in ("det_offsets", "det_ids", "obs_offsets", "obs_ids",
                                                                   "probs"))) for r in range(world)])
    if timings is not None:
        timings.update(shard_s=t1 - t0, exchange_s=t2 - t1, merge_s=t3 - t2, gather_s=time.perf_counter() - t3,
                       merged_entries=int(sum(p[0].numel() for p in mine)))
    return out

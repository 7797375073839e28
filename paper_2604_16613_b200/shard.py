"""Multi-GPU compile of ONE circuit by fault-range sharding.

Rank k of n runs gp_compile_shard on its GPU: the walk (Alg. 1, stepg.cpp)
of every detector word down to the shard's first layer only, and the
emission of the error sources placed in layers [l*k/n, l*(k+1)/n) -- their
noise ops and the outcome flips of their measurements. The result is a
partial table of UNFOLDED signatures (one entry per nonempty source), so the
exchange ships constituent probabilities and the final fold is bit-exact
(dem.cpp:97-106 folds a group's sorted member probabilities).

The one exchange step is a variable-size all-gather of the partial tables
(NCCL over NVLink on GPUs; gloo in the CPU tests); the merge
(gp_merge_partials: bucket / group / fold / write on the device) runs on the
root, or on every rank with ``root=None``. The reference has no multi-GPU
path ("multi-GPU: none in the paper"); the result equals
demc::compile_circuit (compile.cpp:23-53) of the whole circuit.

Arrays travel bit-exactly: u32 as int32, u64 as int64 views, f64 as is.
"""

from __future__ import annotations

import numpy as np

from .api import CorrelationLevel, Dem, PartialTable  # noqa: F401

_WIRE = {np.dtype(np.uint32): np.int32, np.dtype(np.uint64): np.int64, np.dtype(np.int32): np.int32,
         np.dtype(np.int64): np.int64, np.dtype(np.float64): np.float64}


def gather_flat(arrays: dict, device: str, group=None) -> dict:
    """All-gathers variable-length flat arrays: per array one all_gather of
    the lengths, then one of the payloads padded to the longest. Returns
    {name: [per-rank np.ndarray]} on every rank, dtypes preserved bit-exactly."""
    import torch
    import torch.distributed as td

    ws = td.get_world_size(group)
    out = {}
    for name, a in arrays.items():
        a = np.ascontiguousarray(a)
        wire = _WIRE[a.dtype]
        t = torch.from_numpy(a.view(wire)).to(device)
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


def gather_tensors(tensors: dict, group=None) -> dict:
    """Device-resident variant of gather_flat: torch tensors (any device the
    backend supports) all-gathered as {name: [per-rank tensor]} -- over NCCL
    the tables move HBM to HBM over NVLink, never through the host."""
    import torch
    import torch.distributed as td

    ws = td.get_world_size(group)
    out = {}
    for name, t in tensors.items():
        t = t.contiguous()
        n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
        sizes = [torch.zeros_like(n) for _ in range(ws)]
        td.all_gather(sizes, n, group=group)
        lens = [int(x.item()) for x in sizes]
        pad = torch.zeros(max(max(lens), 1), dtype=t.dtype, device=t.device)
        pad[:t.numel()] = t
        parts = [torch.empty_like(pad) for _ in range(ws)]
        td.all_gather(parts, pad, group=group)
        out[name] = [parts[r][:lens[r]] for r in range(ws)]
    return out


def compile_sharded(compiler, circuit, level=CorrelationLevel.L0, group=None, root: int | None = 0) -> Dem | None:
    """One circuit compiled across the ranks of `group` (torch.distributed
    initialised; one process per GPU, compiler on that GPU). Over NCCL the
    partial tables stay in HBM (compile_shard(on_device=True), NVLink
    all-gather, merge from device memory); over gloo they go through the
    host. Returns the DEM on `root` (every rank when root is None), None
    elsewhere."""
    import torch.distributed as td

    from .api import DevicePartialTable

    rank, world = td.get_rank(group), td.get_world_size(group)
    if td.get_backend(group) == "nccl":
        part = compiler.compile_shard(circuit, rank, world, level, on_device=True)
        g = gather_tensors(part.arrays(), group)
        tables = [DevicePartialTable(part.num_detectors, part.num_observables, g["probs"][r], g["rec_offsets"][r],
                                     g["rec_words"][r], g["rec_bits"][r]) for r in range(world)]
    else:
        part = compiler.compile_shard(circuit, rank, world, level)
        tables = tables_from(gather_flat(table_arrays(part), "cpu", group))
    if root is not None and rank != root:
        return None
    return compiler.merge_partials(tables)

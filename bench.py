"""Benchmark of the B200 DEM compile path (driver contract: one JSON line).

Workload (default, config 5 of BASELINE.json): adaptive-branch circuits of the
BB [[72,12,6]] code, 6 rounds, compiled at L0. Each rank owns its own
--branches circuits (branch ids rank*B .. rank*B+B-1, weak scaling); a step
compiles the rank's whole batch. No collective on the data path.

  value  hyperedges/s with inputs resident in HBM: the device pipeline replayed
         K times on the uploaded batch (gp_replay), CUDA-event timed, max over
         ranks. The batch image is larger than L2 (noted in config).
  e2e    the same metric through the public batch API (gp_compile_batch): host
         circuits -> pinned staging -> H2D -> kernels -> D2H of the flat DEM,
         every step; wall-timed around a barrier + synchronize.

--impl reference times the reference CPU compiler (oracle/_ref, built from the
reference sources) on the box's host cores with a std::thread pool (the
demc_main.cpp:184-195 pattern) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "hyperedges/sec and p50 DEM compile latency (ms) at 1/2/4/8 B200 vs CPU ref"
OPT_PIPELINE = 4  # include/greenpeas.h GP_OPT_PIPELINE
UNIT = "hyperedges/s"
WORKLOAD = "bb72_adaptive_branches_r6_L0"
GOLDEN_BRANCHES = ROOT / "tests" / "golden" / "bb72_branches_r6_L0.npz"
L2_BYTES = 126 * 2**20


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Dist:
    def __init__(self, gpus: int, backend: str):
        self.ws, self.rank, self.local = dist_env()
        self.pg = None
        if self.ws > 1:
            import torch
            import torch.distributed as td
            if backend == "nccl":
                torch.cuda.set_device(self.local)
            td.init_process_group(backend=backend)
            self.td, self.torch = td, torch
            self.pg = True
        self.backend = backend

    def barrier(self):
        if self.pg:
            if self.backend == "nccl":
                self.td.barrier(device_ids=[self.local])
            else:
                self.td.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        dev = f"cuda:{self.local}" if self.backend == "nccl" else "cpu"
        t = self.torch.tensor([float(x)], dtype=self.torch.float64, device=dev)
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.pg:
            return x
        dev = f"cuda:{self.local}" if self.backend == "nccl" else "cpu"
        t = self.torch.tensor([float(x)], dtype=self.torch.float64, device=dev)
        self.td.all_reduce(t, op=self.td.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.pg:
            self.td.destroy_process_group()


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        rows = [r.split(",") for r in Path(self.f.name).read_text().splitlines() if r.count(",") >= 8]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def shard(rank: int, world: int, per_rank: int) -> range:
    """Branch ids owned by a rank (weak scaling: every rank owns per_rank)."""
    return range(rank * per_rank, (rank + 1) * per_rank)


def gather_flat(dist, arrays: dict, device: str):
    """Gathers variable-length flat DEM arrays (per-rank tables) to rank 0:
    the final exchange step of SURVEY.md 8e (paper_2604_16613_b200.shard:
    sizes all-gathered, payloads by grouped sends / receives into exact-size
    buffers). Returns {name: [per-rank np.ndarray]} on rank 0, None elsewhere."""
    from paper_2604_16613_b200.shard import gather_to_root
    return gather_to_root(arrays, device, 0)


def build_branches(first: int, count: int):
    import paper_2604_16613_b200 as gp
    return [gp.gen_bb72_branch(first + b) for b in range(count)]


def views_of(circuits):
    from paper_2604_16613_b200 import _native as N
    arr = (N.CircuitView * len(circuits))()
    for i, c in enumerate(circuits):
        arr[i] = c.view()[0]
    return arr


def reference_pool(circuits_text: list[str], level: int, threads: int):
    """Reference compile_circuit on a thread pool; returns (edges, wall_s)."""
    from oracle.bindings import RefLib
    ref = RefLib()
    handles = [ref.parse(t) for t in circuits_text]
    edges, ns = ref.compile_pool(handles, level, threads)
    return edges, ns / 1e9


def cpu_info():
    model = "unknown"
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model, os.cpu_count() or 1


def run_reference(args, dist):
    """--impl reference: rank 0 times the reference CPU compiler on the GPU
    arm's per-GPU workload -- the same args.branches branch circuits (ids
    0..B-1), every step -- on a std::thread pool of all host cores (the
    demc_main.cpp:184-195 pattern). This process loads oracle/_ref/
    libdemc_ref.so only: the branch circuits come from the repo's generator
    source compiled into that library and reach the reference as text through
    its own parse_circuit (oracle/ref_capi.cpp)."""
    if dist.rank != 0:
        return
    from oracle.bindings import RefLib
    ref = RefLib()
    threads = os.cpu_count() or 1
    B = args.branches
    t0 = time.time()
    handles = ref.gen_bb72_branches(0, B, threads=threads)
    gen_s = time.time() - t0
    times, edges = [], 0
    for i in range(args.warmup + args.steps):
        e, ns = ref.compile_pool(handles, args.level, threads)
        if i >= args.warmup:
            times.append(ns / 1e9)
            edges = e
    wall = statistics.mean(times)
    value = edges / wall
    model, ncpu = cpu_info()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64+f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "branches_per_gpu": B, "level": args.level,
                   "hyperedges_per_step": int(edges), "generate_s": round(gen_s, 2),
                   "note": "each step compiles the GPU arm's per-GPU branch set (ids 0..B-1) in full"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"all {B} BB72 r6 branch circuits per step, reference compile_circuit "
                                   f"on a std::thread pool of {threads}", "cpu": model},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit_line(line)


def shim_lib():
    """libgp_shimbench.so: timing harness of the C++ drop-in endpoint
    (demc::compile_circuit -> owning demc::Dem, csrc/gp_shimbench.cpp)."""
    import ctypes as C

    from paper_2604_16613_b200 import _native as N
    L = C.CDLL(str(N.LIB_PATH.parent / "libgp_shimbench.so"))
    L.sb_time_shim.argtypes = [C.POINTER(N.CircuitView), C.c_int, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint64)]
    L.sb_time_shim.restype = C.c_int64
    L.sb_shim_pool.argtypes = [C.POINTER(N.CircuitView), C.c_uint32, C.c_int, C.c_uint32, C.c_uint32,
                               C.POINTER(C.c_uint64)]
    L.sb_shim_pool.restype = C.c_int64
    return L


def pct(ts, q):
    ts = sorted(ts)
    return float(ts[min(len(ts) - 1, int(len(ts) * q))])


def single_circuit_block(compiler, ref_ok: bool, quick: bool, gpu_iters: int, ref_iters: int):
    """N=1 extras (SURVEY 8d timing protocol): p50 compile latency of the
    single-circuit configs 1-4 at both GPU endpoints -- the flat pinned DEM
    (gp_compile) and the owning demc::Dem of the reference signature (the C++
    shim) -- over >= 1,000 compiles each after warm-up, with the reference
    CPU compiler's p50 (1 thread, >= 20 compiles after 1 warm-up,
    demc_main.cpp:126) on the same circuit."""
    import ctypes as C

    import paper_2604_16613_b200 as gp
    cases = [("surface_d3_r3_paper", lambda: gp.gen_surface(3, 3, 1e-3), (0, 2)),
             ("surface_d11_r11_si1000", lambda: gp.gen_surface(11, 11, 1e-3, gp.NOISE_MODEL_SI1000), (0, 2)),
             ("bb144_r12_uniform_depth8", lambda: gp.gen_bb144(12, 1e-3), (0, 2)),
             ("surface_d25_r25_paper", lambda: gp.gen_surface(25, 25, 1e-3), (0,))]
    out = {}
    ref = None
    if ref_ok:
        from oracle.bindings import RefLib
        ref = RefLib()
    shim = shim_lib()
    for name, make, levels in cases:
        g = make()
        text = g.to_text() if ref else None
        view = g.view()[0]
        for lv in levels:
            for _ in range(20):
                dem = compiler.compile(g, lv)
            ts, ks = [], []
            for _ in range(gpu_iters):
                dem = compiler.compile(g, lv)
                ts.append(compiler.last_stats["total_ns"])
                ks.append(compiler.last_stats["kernel_ns"])
            p50 = pct(ts, 0.5) / 1e6
            sns = (C.c_uint64 * gpu_iters)()
            se = shim.sb_time_shim(C.byref(view), lv, 20, gpu_iters, sns)
            s50 = pct(list(sns), 0.5) / 1e6
            # serialize_dem (dem.cpp:144-157) of the DEM: gp_serialize_dem (host, std::to_chars)
            from paper_2604_16613_b200 import _native as N
            dv, keep = dem.view()
            sz = C.c_size_t()
            zs = []
            for _ in range(30):
                t0 = time.perf_counter_ns()
                ptxt = N.lib().gp_serialize_dem(C.byref(dv), C.byref(sz))
                zs.append(time.perf_counter_ns() - t0)
                N.lib().gp_free(ptxt)
            entry = {"edges": dem.num_edges, "iters": gpu_iters, "p50_ms": p50, "p99_ms": pct(ts, 0.99) / 1e6,
                     "serialize_p50_ms": pct(zs, 0.5) / 1e6, "text_bytes": int(sz.value),
                     "kernel_p50_ms": pct(ks, 0.5) / 1e6, "hyperedges_per_s": dem.num_edges / (p50 / 1e3),
                     "dem_endpoint_p50_ms": s50, "dem_endpoint_p99_ms": pct(list(sns), 0.99) / 1e6,
                     "dem_endpoint_ok": int(se) == dem.num_edges}
            if ref is not None and not (quick and "d25" in name):
                e, ns = ref.parse(text).time_compile(lv, ref_iters)
                rp50 = pct(list(ns), 0.5) / 1e6
                _, rz = ref.parse(text).time_serialize(lv, 5 if "d25" in name else 20)
                entry["ref_serialize_p50_ms"] = pct(list(rz), 0.5) / 1e6
                entry.update({"ref_iters": ref_iters, "ref_p50_ms": rp50, "ref_hyperedges_per_s": e / (rp50 / 1e3),
                              "speedup_p50": rp50 / p50, "speedup_p50_dem_endpoint": rp50 / s50})
            out[f"{name}_L{lv}"] = entry
    return out


def link_bandwidths(device: int) -> dict:
    """Measured ceilings of the end-to-end path (GB/s): pinned H2D and D2H
    copies (256 MiB, best of 5, CUDA events) and host memory copy bandwidth
    (torch CPU copy on all threads, best of 3)."""
    import torch
    n = 256 << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=f"cuda:{device}")
    h.fill_(1)
    out = {}
    for name, dst, src in (("h2d_gbs", d, h), ("d2h_gbs", h, d)):
        best = 0.0
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            dst.copy_(src, non_blocking=True)
            b.record()
            b.synchronize()
            best = max(best, n / (a.elapsed_time(b) * 1e6))
        out[name] = best
    x = torch.empty(1 << 30, dtype=torch.uint8)
    y = torch.empty_like(x)
    x.fill_(3)
    best = 0.0
    for _ in range(3):
        t = time.perf_counter()
        y.copy_(x)
        best = max(best, 2 * x.numel() / ((time.perf_counter() - t) * 1e9))
    out["host_copy_gbs"] = best
    out["host_threads"] = torch.get_num_threads()
    del h, d, x, y
    return out


def branch_parity(compiler, out, first: int, count: int, dist) -> dict:
    """Every branch DEM of `out` against the reference's digests
    (tests/golden/bb72_branches_r6_L0.npz: reference hyperedge count and
    gp_dem_digest of its demc::Dem, per branch id); summed over ranks."""
    import numpy as np
    z = np.load(GOLDEN_BRANCHES)
    got = compiler.batch_digests(out)
    eoff = np.ctypeslib.as_array(out.edge_offsets, shape=(count + 1,))
    checked = mism = 0
    if first + count <= len(z["digests"]):
        bad = (got != z["digests"][first:first + count]) | (np.diff(eoff) != z["edges"][first:first + count])
        checked, mism = count, int(np.count_nonzero(bad))
    return {"branches": int(dist.sum(checked)), "mismatches": int(dist.sum(mism)),
            "distinct_dems": int(dist.sum(len(np.unique(got)))),
            "how": "per-branch gp_dem_digest (ids + fp64 bits) == the reference's digest of its own demc::Dem"}


def circuit_bytes(views) -> int:
    """Bytes of the host circuit arrays the packer reads (gp_circuit_view)."""
    total = 0
    for v in views:
        G = v.gate_offsets[v.num_layers]
        Nn = v.noise_offsets[v.num_layers]
        total += 21 * G + 17 * Nn + 8 * (v.num_layers + 1)
        total += 4 * (v.num_detectors + 1 + v.det_offsets[v.num_detectors])
        total += 4 * (v.num_observables + 1 + v.obs_offsets[v.num_observables])
    return total


def sharded_single_block(compiler, dist, reps: int = 10):
    """one large circuit (surface d25 r25, L0) compiled across
    the ranks by fault-range sharding -- shard compile into device tables,
    all-to-all of the entries by owning rank (NCCL send/recv), each owner
    folds its signatures, owners' DEMs gathered to rank 0 -- wall p50 (max
    over ranks) with its phases, the one-GPU compile of the same circuit
    beside it and the merged DEM checked byte for byte against it."""
    import socket

    import torch.distributed as td

    import paper_2604_16613_b200 as gp
    from paper_2604_16613_b200.shard import compile_sharded
    if not td.is_initialized():  # N = 1 (--sharded): a one-rank NCCL group
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        td.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    g = gp.gen_surface(25, 25, 1e-3)
    for _ in range(3):
        compile_sharded(compiler, g, 0)
    ts = []
    phases = {}
    dem = None
    for _ in range(reps):
        dist.barrier()
        t = time.perf_counter()
        tm = {}
        dem = compile_sharded(compiler, g, 0, timings=tm)
        dist.barrier()
        ts.append(dist.max(time.perf_counter() - t))
        for k, v in tm.items():
            phases.setdefault(k, []).append(dist.max(float(v)))
    out = {"circuit": "surface_d25_r25_paper_L0", "shards": max(dist.ws, 1),
           "p50_ms": statistics.median(ts) * 1e3,
           "phases_p50_max_over_ranks": {k: statistics.median(v) * (1e3 if k.endswith("_s") else 1)
                                         for k, v in phases.items()}}
    if dist.rank == 0:
        whole = compiler.compile(g, 0)
        tw = []
        for _ in range(reps):
            t = time.perf_counter()
            compiler.compile(g, 0)
            tw.append(time.perf_counter() - t)
        out["one_gpu_p50_ms"] = statistics.median(tw) * 1e3
        out["identical"] = dem.to_text() == whole.to_text()
        out["edges"] = dem.num_edges
    return out


def run_gpu(args, dist):
    import numpy as np

    import paper_2604_16613_b200 as gp

    ws, rank = dist.ws, dist.rank
    device = dist.local if ws > 1 else 0
    compiler = gp.Compiler(device)
    B = args.branches
    t_gen = time.time()
    circuits = build_branches(shard(rank, ws, B).start, B)
    views = views_of(circuits)
    gen_s = time.time() - t_gen

    # Warm-up through the public API (allocations, first-touch of pinned arenas).
    # The device-resident replay (value) runs the whole batch as one device
    # pass: pipelining off for these compiles.
    compiler.set_option(OPT_PIPELINE, 0)
    for _ in range(args.warmup):
        out, stats = compiler.compile_batch_raw(views, args.level)
    first = shard(rank, ws, B).start
    parity_value_path = branch_parity(compiler, out, first, B, dist) if args.level == 0 else None
    edges = int(out.num_edges)
    h2d = int(stats["h2d_bytes"])
    d2h = int(stats["d2h_bytes"])
    image_bytes = h2d

    # --- value: device-resident replay, CUDA events, max over ranks ---------
    flush = image_bytes < 2 * L2_BYTES
    clocks = Clocks(device)  # sampled across both timed regions
    time.sleep(1.5)  # nvidia-smi start-up
    compiler.replay(args.warmup, flush)
    dist.barrier()
    rep = compiler.replay(args.steps, flush)
    dist.barrier()
    prof = compiler.profile_stages()
    dev_s = dist.max(rep["kernel_ns"] / 1e9)
    total_edges = dist.sum(edges)
    value = total_edges * args.steps / dev_s
    ms_per_step = dev_s / args.steps * 1e3
    launches_per_step = int(rep["kernel_launches"])

    # --- e2e: public batch API, host in / host out, every step ---------------
    # Default (auto) pipelining: sub-batches overlap host packing, upload,
    # device work and the download. Warm-up first (learns output sizes).
    compiler.set_option(OPT_PIPELINE, -1)
    for _ in range(args.warmup):
        compiler.compile_batch_raw(views, args.level)
    dist.barrier()
    t0 = time.perf_counter()
    e2e_parts = {"pack_upload_lower_ms": 0.0, "kernels_ms": 0.0, "download_ms": 0.0}
    for _ in range(args.steps):
        out, stats = compiler.compile_batch_raw(views, args.level)
        e2e_parts["pack_upload_lower_ms"] += stats["lower_ns"] / 1e6 / args.steps
        e2e_parts["kernels_ms"] += stats["kernel_ns"] / 1e6 / args.steps
        e2e_parts["download_ms"] += stats["d2h_ns"] / 1e6 / args.steps
    t1 = time.perf_counter()
    dist.barrier()
    clk = clocks.stop()
    e2e_s = dist.max(t1 - t0)
    e2e_value = total_edges * args.steps / e2e_s
    # parity of the last e2e step's DEMs (the pipelined public-API output)
    parity = branch_parity(compiler, out, first, B, dist) if args.level == 0 else None
    e2e_h2d, e2e_d2h = int(stats["h2d_bytes"]), int(stats["d2h_bytes"])

    # --- device-generated branches: seeds in, DEM out ------
    # gp_compile_bb_branches builds the same branch circuits on the GPU from
    # (seed, branch id): no host circuits, packing or circuit upload; the
    # timed step ends with the batch DEM in host memory, as e2e's does.
    device_gen = None
    if args.level == 0:
        spec = gp.bb72_branch_spec()
        for _ in range(args.warmup):
            out_g, st_g = compiler.compile_bb_branches_raw(spec, first, B, 0)
        dist.barrier()
        g0 = time.perf_counter()
        for _ in range(args.steps):
            out_g, st_g = compiler.compile_bb_branches_raw(spec, first, B, 0)
        g1 = time.perf_counter()
        dist.barrier()
        gen_s = dist.max(g1 - g0)
        device_gen = {"value": total_edges * args.steps / gen_s, "unit": UNIT, "ms_per_step": gen_s / args.steps * 1e3,
                      "h2d_bytes_per_step": int(st_g["h2d_bytes"]), "d2h_bytes_per_step": int(st_g["d2h_bytes"]),
                      "parity": branch_parity(compiler, out_g, first, B, dist),
                      "how": "gp_compile_bb_branches(spec, first branch, count): check subsets drawn and the "
                             "circuits written on the GPU, then the same pipeline; wall time per call, host DEM out"}

    # --- optional final gather of per-rank DEM tables over NCCL -------------
    gather = None
    if ws > 1:
        from paper_2604_16613_b200 import _native as N
        E_ = int(out.num_edges)
        doff_ = N.copy_u32(out.det_offsets, E_ + 1)
        arrays = {"edge_offsets": N.copy_u64(out.edge_offsets, len(circuits) + 1), "det_offsets": doff_,
                  "det_ids": N.copy_u32(out.det_ids, int(doff_[-1])), "probs": N.copy_f64(out.probs, E_)}
        dist.barrier()
        g0 = time.perf_counter()
        got = gather_flat(dist, arrays, f"cuda:{device}")
        dist.barrier()
        gms = dist.max(time.perf_counter() - g0) * 1e3
        if rank == 0:
            gather = {"ms": gms, "to": "rank 0 (grouped NCCL send/recv)",
                      "bytes": int(sum(sum(x.nbytes for x in v) for v in got.values())),
                      "edges": int(sum(len(x) for x in got["probs"]))}

    # --- roofline of the dominant kernel ------------------------------------
    from paper_2604_16613_b200 import _native as N
    E = int(out.num_edges)
    eoff = N.copy_u64(out.edge_offsets, len(circuits) + 1)
    doff = N.copy_u32(out.det_offsets, E + 1).astype(np.int64)
    ooff = N.copy_u32(out.obs_offsets, E + 1).astype(np.int64)
    ab = {"traverse": 0, "reduce": 0, "total": 0}
    for i, c in enumerate(circuits):  # B_alg is per circuit; sum over the batch
        e0, e1 = int(eoff[i]), int(eoff[i + 1])
        ids = int(doff[e1] - doff[e0] + ooff[e1] - ooff[e0])
        for k, v in gp.algorithmic_bytes(gp.circuit_metrics(c, args.level), e1 - e0, ids).items():
            ab[k] += v
    stages = {k: v / args.steps for k, v in prof.items()}
    # Dominant device stage: the traversal (Alg. 1 + fused signature emission)
    # or the reduce (key .. write); achieved = its SURVEY 8d algorithmic bytes
    # over its live CUDA-event time.
    trav_ns = stages.get("traverse", 0) + stages.get("emit", 0)
    red_keys = ("key", "scan_bucket", "scatter", "bucket", "scan_out", "write")
    red_ns = sum(stages.get(k, 0) for k in red_keys)
    part = "traverse" if trav_ns >= red_ns else "reduce"
    dom_ns = trav_ns if part == "traverse" else red_ns
    dominant = "traverse_kernel" if part == "traverse" else "reduce (" + "+".join(red_keys) + ")"
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    achieved = ab[part] / dom_ns if dom_ns else 0.0  # bytes/ns == GB/s
    traffic = None  # ncu dram bytes per launch of the dominant stage, same workload (profiles/)
    tpath = ROOT / "profiles" / "traffic.json"
    if tpath.exists():
        traffic = json.loads(tpath.read_text()).get(part)
    roofline = {"bound": "hbm", "kernel": dominant, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "alg_bytes_per_launch": ab[part], "bytes_per_hyperedge": ab["total"] / max(E, 1),
                "stage_ms": {k: v / 1e6 for k, v in stages.items()},
                "pipeline_alg_gbs": ab["total"] / (rep["kernel_ns"] / args.steps)}
    if args.ncu_traffic is not None:
        roofline["traffic"] = args.ncu_traffic

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64+f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "branches_per_gpu": B, "total_branches": B * ws,
                   "code": "BB [[72,12,6]], Bravyi et al. depth-8 syndrome cycle (7 CX layers; X prep/measure "
                           "as R/MR + H), paper noise NoiseModel{1e-3}, 6 rounds, checks of non-full rounds "
                           "kept with probability 1/2 (mt19937_64 seed_seq{1,0,b,0})",
                   "level": args.level, "hyperedges_per_step": int(total_edges),
                   "parallelism": f"branch-sharded x{ws}, no collective",
                   "l2": "inputs larger than L2" if not flush else "L2 flushed between timed iterations",
                   "input_image_bytes_per_gpu": image_bytes, "generate_s": round(gen_s, 2)},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": e2e_h2d, "d2h_bytes_per_step": e2e_d2h,
                "ms_per_step": e2e_s / args.steps * 1e3, "breakdown": e2e_parts},
        "parity": parity,
        "parity_value_path": parity_value_path,
        "device_generated": device_gen,
        "gpu_launches": launches_per_step * args.steps,
        "gather": gather,
        "roofline": roofline,
        "clocks": clk,
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        model, ncpu = cpu_info()
        sample = args.cpu_sample
        texts = [circuits[b].to_text() for b in range(min(sample, B))]
        threads = ncpu
        e, wall = reference_pool(texts, args.level, threads)
        line["cpu_baseline"] = {"value": e / wall, "unit": UNIT, "cores": threads, "kind": "reference",
                                "sample": f"{len(texts)} of the {B} branch circuits, reference compile_circuit "
                                          f"on a {threads}-thread pool ({wall:.2f} s wall)", "cpu": model}
    # e2e roof: what the host <-> device path allows per step, from measured
    # link and host-memory bandwidths (pipelined: the stages overlap, so the
    # floor is the slowest of them)
    bw = link_bandwidths(device)
    in_bytes = circuit_bytes(views)
    roof = {"h2d_ms": e2e_h2d / (bw["h2d_gbs"] * 1e6), "d2h_ms": e2e_d2h / (bw["d2h_gbs"] * 1e6),
            "host_ms": (in_bytes + e2e_h2d + e2e_d2h) / (bw["host_copy_gbs"] * 1e6), "device_ms": ms_per_step,
            "input_circuit_bytes": in_bytes, **bw}
    roof["bound_ms"] = max(roof["h2d_ms"], roof["d2h_ms"], roof["host_ms"], roof["device_ms"])
    roof["e2e_ms"] = e2e_s / args.steps * 1e3
    roof["frac"] = roof["bound_ms"] / roof["e2e_ms"]
    roof["how"] = ("host_ms = (circuit arrays read + staging image written + DEM written to pinned memory) / "
                   "host copy bandwidth; h2d/d2h = bytes / pinned-copy bandwidth; device_ms = value's ms/step")
    line["e2e"]["roof"] = roof
    if rank == 0 and ws == 1 and not args.no_single:
        line["single_circuit"] = single_circuit_block(compiler, ref_ok=not args.no_cpu_baseline, quick=args.quick,
                                                      gpu_iters=args.gpu_iters, ref_iters=args.ref_iters)
    if rank == 0 and ws == 1 and not args.no_shim_pool:
        import ctypes as C
        wall = C.c_uint64()
        thr = os.cpu_count() or 1
        e = shim_lib().sb_shim_pool(views, B, args.level, thr, 3, C.byref(wall))
        line["dem_endpoint_pool"] = {
            "value": e / (wall.value / 1e9) if e > 0 else None, "unit": UNIT, "threads": thr, "circuits": B,
            "ms_per_pass": wall.value / 1e6,
            "how": "demc_main.cpp:184-195 pattern over the C++ drop-in: host threads, atomic counter, one "
                   "demc::compile_circuit(c, L0, 1) per branch (one GPU context per thread, shared packing pool)"}
    if ws > 1 or args.sharded:
        try:
            blk = sharded_single_block(compiler, dist)
        except Exception as e:  # the headline line must still be printed
            blk = {"error": repr(e)[:300]}
        if rank == 0:
            line["sharded_single"] = blk
    if rank == 0:
        emit_line(line)


_JSON_FD = None


def emit_line(line: dict) -> None:
    """The one JSON line, on the original stdout (everything else -- library
    or NCCL chatter included -- goes to stderr, see main)."""
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)


def main():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)  # fd 1 -> stderr for the rest of the run
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="greenpeas", choices=["greenpeas", "reference"])
    ap.add_argument("--branches", type=int, default=4096, help="branch circuits per GPU")
    ap.add_argument("--level", type=int, default=0)
    ap.add_argument("--cpu-sample", type=int, default=1024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-single", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="also at N=1: fault-range sharded d25 block (over NCCL)")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--gpu-iters", type=int, default=1000, help="single-circuit GPU compiles per case")
    ap.add_argument("--ref-iters", type=int, default=20, help="single-circuit reference compiles per case")
    ap.add_argument("--no-shim-pool", action="store_true")
    ap.add_argument("--ncu-traffic", type=float, default=None)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    ws, _, _ = dist_env()
    dist = Dist(args.gpus, "nccl" if args.impl == "greenpeas" else "gloo") if ws > 1 else Dist(1, "none")
    try:
        if args.impl == "reference":
            run_reference(args, dist)
        else:
            run_gpu(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()

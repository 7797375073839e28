"""The demc_main.cpp:184-195 pattern over the C++ drop-in (developer tool):
host threads taking BB72 r6 branch circuits from a counter, one
demc::compile_circuit each (bench.py's dem_endpoint_pool block, alone).
usage: python tools/shim_pool.py [branches] [threads] [reps]"""
import ctypes as C
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2604_16613_b200 as gp  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
thr = int(sys.argv[2]) if len(sys.argv) > 2 else (os.cpu_count() or 1)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
gens = [gp.gen_bb72_branch(b) for b in range(B)]
views = bench.views_of(gens)
wall = C.c_uint64()
e = bench.shim_lib().sb_shim_pool(views, B, 0, thr, reps, C.byref(wall))
print(f"threads {thr}: {wall.value / 1e6:.1f} ms per pass of {B} circuits, {e / (wall.value / 1e9) / 1e6:.1f} M hyperedges/s")

"""Phase times of the C++ drop-in endpoint (developer tool): flatten of the
demc::Circuit, the compile, and the demc::Dem materialisation, per call
(GP_LAT_TRACE lines from demc_shim.cpp), for the single-circuit configs.
usage: GP_LAT_TRACE=1 python tools/shim_trace.py [iters]"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2604_16613_b200 as gp  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
shim = bench.shim_lib()
for name, g in [("bb144_r12", gp.gen_bb144(12, 1e-3)), ("d25_r25", gp.gen_surface(25, 25, 1e-3)),
                ("d11_si1000", gp.gen_surface(11, 11, 1e-3, gp.NOISE_MODEL_SI1000))]:
    view = g.view()[0]
    for lv in (0, 2) if name != "d25_r25" else (0,):
        ns = (C.c_uint64 * iters)()
        print(f"== {name} L{lv}", file=sys.stderr, flush=True)
        e = shim.sb_time_shim(C.byref(view), lv, 5, iters, ns)
        print(name, lv, e, sorted(ns)[iters // 2] / 1e3, "us p50", flush=True)

"""Single-circuit latency breakdown (developer tool): p50 of gp_compile total
and of each gp_stats component, plus per-stage device times from gp_replay."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_16613_b200 as gp

cases = [("d3_L0", lambda: gp.gen_surface(3, 3, 1e-3), 0),
         ("d11_L0", lambda: gp.gen_surface(11, 11, 1e-3, gp.NOISE_MODEL_SI1000), 0),
         ("d11_L2", lambda: gp.gen_surface(11, 11, 1e-3, gp.NOISE_MODEL_SI1000), 2),
         ("bb144_L0", lambda: gp.gen_bb144(12, 1e-3), 0),
         ("bb144_L2", lambda: gp.gen_bb144(12, 1e-3), 2),
         ("d25_L0", lambda: gp.gen_surface(25, 25, 1e-3), 0)]
only = set(sys.argv[1:])
comp = gp.Compiler(0)
for name, make, lv in cases:
    if only and name not in only:
        continue
    g = make()
    for _ in range(5):
        comp.compile(g, lv)
    rows = []
    iters = 50 if "d25" in name else 200
    for _ in range(iters):
        comp.compile(g, lv)
        rows.append(dict(comp.last_stats))
    med = lambda k: sorted(r[k] for r in rows)[len(rows) // 2] / 1e3
    keys = ["total_ns", "lower_ns", "h2d_ns", "kernel_ns", "traverse_ns", "reduce_ns", "d2h_ns"]
    print(f"{name}: " + " ".join(f"{k[:-3]}={med(k):.1f}us" for k in keys), f"launches={rows[-1]['kernel_launches']}",
          flush=True)
    comp.replay(20)
    st = comp.profile_stages()
    print("   replay stages (us):", " ".join(f"{k}={v / 20 / 1e3:.1f}" for k, v in st.items()), flush=True)

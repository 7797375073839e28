"""Quick GPU parity sweep (developer tool): GPU vs C restatement vs reference."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_16613_b200 as gp
from oracle.bindings import Port, parse_dem_text

port = Port()
comp = gp.Compiler(0)
fails = 0
root = Path(__file__).resolve().parents[1]
for fx in sorted((root / 'tests/golden/fixtures').iterdir()):
    c = gp.parse_circuit((fx / 'circuit.txt').read_text()); lv = int((fx / 'level').read_text())
    got = comp.compile(c, lv).hyperedges()
    exp = parse_dem_text((fx / 'expected.dem').read_text())
    ok = got == exp
    fails += not ok
    print(fx.name, len(got), len(exp), 'OK' if ok else 'MISMATCH', flush=True)
    if not ok:
        print(' got', got[:5]); print(' exp', exp[:5])
cases = [('rep3_2', gp.gen_repetition(3, 2, 1e-3)), ('surf3_3', gp.gen_surface(3, 3, 1e-3)),
         ('surf5_3', gp.gen_surface(5, 3, 1e-3)), ('si1000_5', gp.gen_surface(5, 5, 1e-3, 1)),
         ('bb72_r2', gp.gen_bb(6, 6, rounds=2)), ('branch', gp.gen_bb72_branch(5, rounds=4))]
for name, g in cases:
    c = g.to_circuit()
    for lv in (0, 1, 2):
        got = comp.compile(g, lv).hyperedges()
        exp, _, _ = port.compile(c, lv)
        ok = got == exp
        fails += not ok
        print(name, lv, len(got), len(exp), 'OK' if ok else 'MISMATCH', comp.last_stats['total_ns'] / 1e3, 'us', flush=True)
        if not ok:
            sg, se = set(got), set(exp)
            print(' only gpu', list(sg - se)[:5]); print(' only oracle', list(se - sg)[:5])
# batch
gs = [gp.gen_bb72_branch(b, rounds=4) for b in range(6)]
outs = comp.compile_batch(gs, 0)
for b, (g, d) in enumerate(zip(gs, outs)):
    exp, _, _ = port.compile(g.to_circuit(), 0)
    ok = d.hyperedges() == exp
    fails += not ok
    print('batch', b, d.num_edges, len(exp), 'OK' if ok else 'MISMATCH')
# timing
for name, g, lv in [('bb144 L0', gp.gen_bb144(), 0), ('bb144 L2', gp.gen_bb144(), 2), ('d11 si L2', gp.gen_surface(11, 11, 1e-3, 1), 2)]:
    for _ in range(3):
        d = comp.compile(g, lv)
    ts = []
    for _ in range(20):
        d = comp.compile(g, lv); ts.append(comp.last_stats['total_ns'])
    ts.sort()
    print(name, 'E', d.num_edges, 'p50 us', ts[10] / 1e3, comp.last_stats)
print('FAILS', fails)
sys.exit(1 if fails else 0)

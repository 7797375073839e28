"""Minimal GPU smoke for kernel debugging: fixtures + one batch."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_16613_b200 as gp
from oracle.bindings import Port, parse_dem_text
root = Path(__file__).resolve().parents[1]
comp = gp.Compiler(0)
bad = 0
for fx in sorted((root / 'tests/golden/fixtures').iterdir()):
    c = gp.parse_circuit((fx / 'circuit.txt').read_text()); lv = int((fx / 'level').read_text())
    ok = comp.compile(c, lv).to_text() == (fx / 'expected.dem').read_text()
    bad += not ok
    print(fx.name, ok, flush=True)
port = Port()
gens = [gp.gen_bb72_branch(b, rounds=3) for b in range(400)]
t = time.time(); ds = comp.compile_batch(gens, 0); print('batch', time.time() - t, comp.last_stats, flush=True)
for b in (0, 17, 399):
    ok = ds[b].hyperedges() == port.compile(gens[b].to_circuit(), 0)[0]
    bad += not ok
    print('branch', b, ok, flush=True)
g = gp.gen_bb144()
for lv in (0, 2):
    for _ in range(3): d = comp.compile(g, lv)
    print('bb144', lv, d.num_edges, comp.last_stats, flush=True)
print('BAD', bad)

"""Repro: a batch first, then BB144 compiles on the same context; hashes vs reference."""
import hashlib, json, sys
from pathlib import Path
root = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(root))
import paper_2604_16613_b200 as gp
full = json.loads((root / "tests/golden/full_size.json").read_text())["bb144_r12_uniform"]["levels"]
c = gp.Compiler(0)
if sys.argv[1] == "batch":
    c.compile_batch([gp.gen_bb72_branch(b, rounds=3) for b in range(400)], 0)
g = gp.gen_bb144()
for lv in [int(x) for x in sys.argv[2:]]:
    try:
        d = c.compile(g, lv)
        ok = hashlib.sha256(d.to_text().encode()).hexdigest() == full[str(lv)]["dem_sha256"]
        print(lv, d.num_edges, "OK" if ok else "MISMATCH", c.last_stats["kernel_launches"], flush=True)
    except Exception as e:
        print(lv, "ERR", e, flush=True)
        break

"""Per-kernel SASS evidence of libgreenpeas (developer tool): resource usage
(cuobjdump -res-usage) and counts of the mnemonics that matter here -- bulk
async copies (UBLKCP: cp.async.bulk / the non-tensor TMA path), mbarrier
waits (SYNCS), shared-memory atomics (ATOMS), warp votes / shuffles, fp64 math
-- and the absence of tensor-core instructions (this is GF(2) + fp64 scalar
work). usage: python tools/sass_summary.py [object] > profiles/rNN/sass_summary.txt"""
import re
import subprocess
import sys
from collections import Counter, defaultdict

obj = sys.argv[1] if len(sys.argv) > 1 else "paper_2604_16613_b200/_lib/gp_kernels.o"
res = subprocess.run(["cuobjdump", "-res-usage", obj], capture_output=True, text=True).stdout
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
usage = {}
cur = None
for line in res.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m:
        cur = m.group(1)
    elif cur and "REG:" in line:
        usage[cur] = " ".join(line.split()[:4])
counts = defaultdict(Counter)
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if cur and m:
        counts[cur][m.group(1).split(".")[0]] += 1
keys = ["UBLKCP", "SYNCS", "ATOMS", "ATOMG", "RED", "VOTE", "SHFL", "DFMA", "DMUL", "DADD", "BAR", "HMMA", "UTCMMA",
        "UTCHMMA", "LDS", "STS", "LDG", "STG"]
print(f"# {obj}\n# kernel | resources | instructions | " + " ".join(keys))
for k in sorted(counts):
    c = counts[k]
    name = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()[:90]
    print(f"{name}\n  {usage.get(k, '?')}  total {sum(c.values())}  " + " ".join(f"{x}={c[x]}" for x in keys if c[x]))

"""Instruction / stall share of a kernel by source-line region (developer tool):
python tools/ncu_regions.py report.ncu-rep kernel-regex file:lo-hi=name ..."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
regions = []
for a in sys.argv[3:]:
    loc, name = a.split("=")
    f, rng = loc.split(":")
    lo, hi = map(int, rng.split("-"))
    regions.append((f, lo, hi, name))
out = subprocess.run(["ncu", "-i", rep, "--kernel-name", "regex:" + kern, "--page", "source", "--csv",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, hdr = "?", None
agg = {}
tot_i = tot_s = 0.0
num = lambda x: float(x) if x not in ("", "-") else 0.0
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit() and len(r) == len(hdr):
        ln = int(r[0])
        i, s = num(r[hdr.index("Instructions Executed")]), num(r[hdr.index("Warp Stall Sampling (All Samples)")])
        tot_i += i
        tot_s += s
        key = "other:" + fname
        for f, lo, hi, name in regions:
            if f == fname and lo <= ln <= hi:
                key = name
                break
        a = agg.setdefault(key, [0.0, 0.0])
        a[0] += i
        a[1] += s
for k, (i, s) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:40s} inst {100 * i / max(tot_i, 1):5.1f}%  stall {100 * s / max(tot_s, 1):5.1f}%")

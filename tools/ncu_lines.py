"""Per-source-line hot spots of one kernel in an ncu report (developer tool).
usage: python tools/ncu_lines.py report.ncu-rep [top] [kernel-regex]"""
import csv, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kfilt = ["--kernel-name", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, *kfilt, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, hdr, lines = "?", None, []
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
        lines.append((fname, int(r[0]), r[1], r))
if not lines:
    sys.exit("no per-line metrics in " + rep)
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_e = hdr.index("Instructions Executed")
num = lambda x: float(x) if x not in ("", "-") else 0.0
ts = sum(num(l[3][i_s]) for l in lines) or 1
te = sum(num(l[3][i_e]) for l in lines) or 1
print(f"samples {ts:.0f}  warp-instructions {te:.0f}")
for f, ln, src, r in sorted(lines, key=lambda l: -num(l[3][i_s]))[:top]:
    print(f"{f}:{ln:<5} stall {100 * num(r[i_s]) / ts:5.1f}%  inst {100 * num(r[i_e]) / te:5.1f}%  {src.strip()[:80]}")

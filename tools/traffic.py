"""profiles/traffic.json from an ncu --set full capture of ONE batch compile
(tools/fast_repro.py, the bench workload): DRAM bytes (read + write) per
stage and compile -- 'traverse' (traverse_kernel) and 'reduce' (key .. write
kernels), each kernel averaged over its launches in the capture."""
import csv
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
iK, iR, iW = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
red = ("key_kernel", "scatter_kernel", "bucket_kernel", "huge_kernel", "write_kernel", "scan_")
# per compile: the capture holds several compiles of the same batch (the
# first may be a capacity-learning pass); each kernel's bytes are averaged
# over its launches, and a stage is the sum of its kernels' averages
per, cnt = {}, {}
for r in rows[2:]:
    k = r[iK]
    b = float(r[iR].replace(",", "")) * scale[units[iR]] + float(r[iW].replace(",", "")) * scale[units[iW]]
    name = k.split("(")[0]
    per[name] = per.get(name, 0) + b
    cnt[name] = cnt.get(name, 0) + 1
avg = {k: per[k] / cnt[k] for k in per}
acc = {"traverse": sum(v for k, v in avg.items() if "traverse_kernel" in k),
       "reduce": sum(v for k, v in avg.items() if any(x in k for x in red)),
       "per_kernel": avg, "launches": cnt}
acc["source"] = "ncu --set full, one compile of 4096 BB72 branch circuits (L0), tools/fast_repro.py 4096"
json.dump(acc, open(out, "w"), indent=1)
print(json.dumps(acc, indent=1))

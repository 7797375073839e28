"""Summarise ncu outputs into profiles/: launch-list shares and key metrics."""
import csv, subprocess, sys
from collections import defaultdict


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = r[4].split("(")[0].replace("unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += float(r[-1])
    tot = sum(v[1] for v in agg.values())
    out = [f"{'kernel':40s} {'launches':>8s} {'total_us':>12s} {'mean_us':>10s} {'share':>7s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:40s} {n:8d} {t / 1e3:12.1f} {t / n / 1e3:10.2f} {100 * t / tot:6.1f}%")
    return "\n".join(out)


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread", "launch__grid_size",
           "launch__block_size", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem"]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        out.append(f"kernel: {vals[hdr.index('Kernel Name')][:90]}")
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                out.append(f"  {m:60s} {vals[i]:>16s} {units[i]}")
    sass = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                          text=True).stdout
    rows = list(csv.reader(sass.splitlines()))
    if len(rows) > 2:
        h = rows[1]
        iS = h.index("Warp Stall Sampling (All Samples)")
        cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
        agg = defaultdict(int)
        for r in rows[2:]:
            for i in cols:
                if i < len(r) and r[i].isdigit():
                    agg[h[i]] += int(r[i])
        tot = sum(agg.values()) or 1
        out.append("  warp stall samples: " + ", ".join(f"{k[6:]} {100 * v / tot:.0f}%" for k, v in
                                                       sorted(agg.items(), key=lambda x: -x[1])[:6]))
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"### {p}")
        print(launches(p) if p.endswith(".csv") else report(p))
        print()

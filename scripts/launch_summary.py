"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,... --csv --log-file)
into per-kernel launch counts and median / mean durations (the kernel shares of the
step; cold-cache, serialised launches).
  python scripts/launch_summary.py gpurun_out/r02a/launches.csv > profiles/r02/launches_summary.txt"""
import collections
import csv
import statistics
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
ui = h.index("Metric Unit")
per = collections.defaultdict(dict)
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
    if r[mi] == "gpu__time_duration.sum":
        v *= scale
    per[(int(r[ii]), r[ki])][r[mi]] = v
by = collections.defaultdict(list)
for (i, k), m in per.items():
    by[k].append(m)
tot = 0.0
lines = []
for k, ms in by.items():
    d = [m["gpu__time_duration.sum"] for m in ms if "gpu__time_duration.sum" in m]
    rd = [m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in ms]
    med = statistics.median(d)
    tot += med
    lines.append((med, f"  {k[:70]:70s} n={len(d):4d} median={med:9.1f}us mean={statistics.mean(d):9.1f}us "
                       f"dram_median={statistics.median(rd) / 1e6 if rd else 0:8.1f}MB"))
for _, line in sorted(lines, reverse=True):
    print(line)

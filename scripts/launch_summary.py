"""Summarise an ncu --metrics gpu__time_duration.sum launch list (per kernel: launches,
median and mean us). The bench's list mixes arms (realb / bf16 / fp4all steps, e2e,
roofline launches); in the fp4all steps the BF16 GEMMs have no groups and exit at
once, so the median is the representative figure for a kernel of the headline step."""
import collections, csv, statistics, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows:
    v = float(r[vi].replace(",", ""))
    v = v / 1000 if r[ui] in ("nsecond", "ns") else v * 1000 if r[ui] in ("msecond", "ms") else v
    agg.setdefault(r[ki][:70], []).append(v)
for n, v in agg.items():
    if "realb" in n or "--all" in sys.argv:
        print(f"  {n:70s} n={len(v):3d} median={statistics.median(v):8.1f}us mean={sum(v)/len(v):8.1f}us")

"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per kernel launches, total and mean device time.  python tools/launch_summary.py file.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, data = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
agg = collections.defaultdict(list)
for r in data:
    agg[r[ki].split("(")[0][:48]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    v.sort()
    print(f"{k:48s} n={len(v):5d} total={sum(v) / 1e3:9.3f} ms ({sum(v) / tot:5.1%}) mean={sum(v) / len(v):9.2f} us "
          f"p50={v[len(v) // 2]:9.2f} us max={v[-1]:9.2f} us")

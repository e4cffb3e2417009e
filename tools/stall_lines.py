"""Warp-stall samples per CUDA source line (with the dominant stall reasons)
from `ncu -i REP --page source --csv --print-source cuda,sass` output.
  python tools/stall_lines.py source.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fn, hdr = None, None
agg, src = collections.Counter(), {}
why = collections.defaultdict(collections.Counter)
total_why = collections.Counter()
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fn = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name",) or r[0] == "Line No":
        hdr = r if r[0] == "Line No" else hdr
        continue
    if hdr is None or r[0] == "":
        continue
    d = dict(zip(hdr[4:], r[4:]))  # the source row's metric columns follow the two (sass) columns
    key = (fn, r[0])
    src[key] = r[1][:90]
    try:
        agg[key] += int(r[4])
    except ValueError:
        continue
    for h, v in zip(hdr, r):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                n = int(v)
            except ValueError:
                continue
            if n:
                why[key][h[6:]] += n
                total_why[h[6:]] += n
tot = sum(agg.values()) or 1
print("total samples", tot, "by reason:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in total_why.most_common(8)))
for key, s in agg.most_common(top):
    w = ", ".join(f"{k} {v}" for k, v in why[key].most_common(3))
    print(f"{s:7d} {100 * s / tot:5.1f}% {key[0]}:{key[1]:<5} {src[key]:<90} [{w}]")

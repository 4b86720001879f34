"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel mean time."""
import csv
import sys
from collections import OrderedDict

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    if not rows:
        print(f, "empty"); continue
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = OrderedDict()
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        v = float(r[vi].replace(",", ""))
        if r[ui] == "usecond": v *= 1e3
        if r[ui] == "msecond": v *= 1e6
        agg.setdefault(name, []).append(v)
    print(f)
    tot = sum(sum(v) for v in agg.values())
    for k, v in agg.items():
        print(f"  {k[:48]:48s} n={len(v):4d} mean={sum(v)/len(v)/1e3:9.2f} us  share={sum(v)/tot*100:5.1f}%")

"""Summarise ncu --csv launch lists (one or more metrics per launch).

Per kernel: launch count, mean gpu__time_duration, share of the summed time and,
when captured, mean DRAM bytes (read + write) per launch.

  python tools/launches.py launches.csv [more.csv ...] [--json out.json]
"""
import csv
import json
import sys
from collections import OrderedDict

SCALE = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "KB": 1024.0, "MB": 1024.0 ** 2, "GB": 1024.0 ** 3}


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    if not rows:
        return OrderedDict()
    hdr = rows[0]
    ii, ki = hdr.index("ID"), hdr.index("Kernel Name")
    mi, ui, vi = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    launches = OrderedDict()
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        name = name.replace("unnamed>::", "")
        d = launches.setdefault(r[ii], {"name": name})
        try:
            d[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        except ValueError:
            pass
    return launches


def summarise(launches):
    agg = OrderedDict()
    for d in launches.values():
        a = agg.setdefault(d["name"], {"n": 0, "ns": 0.0, "dram": 0.0, "has_dram": False})
        a["n"] += 1
        a["ns"] += d.get("gpu__time_duration.sum", 0.0)
        if "dram__bytes_read.sum" in d:
            a["has_dram"] = True
            a["dram"] += d["dram__bytes_read.sum"] + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a["ns"] for a in agg.values()) or 1.0
    out = OrderedDict()
    for k, a in agg.items():
        out[k] = {"launches": a["n"], "mean_us": a["ns"] / a["n"] / 1e3,
                  "share": a["ns"] / tot,
                  "dram_bytes_per_launch": a["dram"] / a["n"] if a["has_dram"] else None}
    return out


def main(argv):
    js = None
    if "--json" in argv:
        i = argv.index("--json")
        js = argv[i + 1]
        argv = argv[:i] + argv[i + 2:]
    allres = {}
    for f in argv:
        s = summarise(load(f))
        allres[f] = s
        print(f)
        if not s:
            print("  empty")
        for k, a in s.items():
            dram = (f"  dram={a['dram_bytes_per_launch'] / 1e6:9.3f} MB"
                    if a["dram_bytes_per_launch"] is not None else "")
            print(f"  {k[:44]:44s} n={a['launches']:5d} mean={a['mean_us']:9.2f} us "
                  f"share={a['share'] * 100:5.1f}%{dram}")
    if js:
        with open(js, "w") as f:
            json.dump(allres, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])

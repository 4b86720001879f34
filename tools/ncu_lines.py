"""Per-source-line warp-stall and instruction shares of one kernel in an ncu report.
  python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kre}", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
si, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
te = hdr.index("Thread Instructions Executed")
agg = defaultdict(lambda: [0.0, 0.0, 0.0])
src, cur = {}, None
for r in rows:
    if len(r) < len(hdr) or r[0] == "Line No":
        continue
    if r[0].strip():
        try:
            cur = int(r[0])
            src[cur] = r[1]
        except ValueError:
            pass
    try:
        agg[cur][0] += float(r[si] or 0)
        agg[cur][1] += float(r[ie] or 0)
        agg[cur][2] += float(r[te] or 0)
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
print(f"warp inst {toti:.3e}  thread inst/warp inst {sum(v[2] for v in agg.values()) / toti:.1f}")
for ln, (a, b, c) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{ln}: stall {a / tot * 100:5.1f}%  inst {b / toti * 100:5.1f}%  "
          f"thr/inst {c / max(b, 1):4.1f}  {src.get(ln, '').strip()[:70]}")

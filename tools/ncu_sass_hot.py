"""Hot SASS instructions + aggregate stall reasons of one kernel in an ncu report.
  python tools/ncu_sass_hot.py report.ncu-rep kernel_regex [launch_skip] [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", f"regex:{kre}", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
si = hdr.index("Warp Stall Sampling (All Samples)")
stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[si] or 0) for r in data)
agg = {hdr[i]: sum(float(r[i] or 0) for r in data) for i in stalls}
print(rows[0][1][:120])
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
    print(f"  {k:28s} {v / tot * 100:5.1f}%")
print("hot instructions:")
for idx, r in sorted(enumerate(data), key=lambda x: -float(x[1][si] or 0))[:top]:
    top_st = sorted(((hdr[i], float(r[i] or 0)) for i in stalls), key=lambda x: -x[1])[:2]
    print(f"  #{idx:5d} {float(r[si]) / tot * 100:5.1f}%  {r[1].strip()[:60]:60s} "
          + " ".join(f"{n[6:]}={v:.0f}" for n, v in top_st))

"""Summarise ncu --set full reports: duration, DRAM bytes, throughputs, occupancy, top stalls."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__inst_executed.sum", "l1tex__t_bytes.sum"]
for path in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        print(path, "no data"); continue
    h, units = rows[0], rows[1]
    print(f"== {path}")
    for r in rows[2:]:
        name = r[h.index("Kernel Name")][:60]
        print(f"  kernel {name}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"    {k:60s} {r[i]:>14s} {units[i]}")
        stalls = [(float(r[i].replace(',', '') or 0), n) for i, n in enumerate(h)
                  if n.startswith("smsp__average_warp_latency_issue_stalled_") and n.endswith(".ratio")
                  and r[i].replace(',', '').replace('.', '').isdigit()]
        stalls.sort(reverse=True)
        for v, n in stalls[:5]:
            print(f"    stall {n.replace('smsp__average_warp_latency_issue_stalled_', ''):48s} {v:8.2f}")

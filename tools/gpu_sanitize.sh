#!/bin/bash
# compute-sanitizer over tools/sanitize_kernels.py (one gpurun call); logs in gpurun_out/
O=gpurun_out; mkdir -p $O
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_kernels.py > $O/san_$tool.log 2>&1
  echo "== $tool: $(grep -h 'sanitize workload' $O/san_$tool.log | tail -1) $(grep -h 'SUMMARY' $O/san_$tool.log | tail -1)"
done
SLCS_NO_FUSED_REACH=1 timeout 1500 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_kernels.py > $O/san_racecheck_tiled.log 2>&1
echo "== racecheck_tiled: $(grep -h 'sanitize workload' $O/san_racecheck_tiled.log | tail -1) $(grep -h 'SUMMARY' $O/san_racecheck_tiled.log | tail -1)"

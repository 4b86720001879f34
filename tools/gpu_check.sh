#!/bin/bash
# one gpurun call: parity tests, race stress, per-kernel launch profile
set -o pipefail
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 200 python tools/debug_ccl.py 2>&1 | tail -3
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_blob.csv timeout 200 python tools/prof_primitives.py --reps 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rand.csv timeout 200 python tools/prof_primitives.py --reps 2 --random 0.5 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_blob.csv gpurun_out/launches_rand.csv

#!/bin/bash
# one gpurun call: parity tests, bench, per-kernel launch profiles (4096 blob, 16384 random)
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -c 1800 gpurun_out/bench.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_blob.csv timeout 200 python tools/prof_primitives.py --reps 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r16k.csv timeout 300 python tools/prof_primitives.py --reps 1 --random 0.5 --size 16384 --ops reach,ccl > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_blob.csv gpurun_out/launches_r16k.csv

#!/bin/bash
# CCL/reach/maxvol iteration: parity subset, C4/C5 bench lines, per-kernel times at 16384^2
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_ccl_gpu.py tests/test_reach_gpu.py tests/test_bands_gpu.py tests/test_executor_gpu.py tests/test_concurrency_gpu.py tests/test_host_pinned_gpu.py tests/test_large_parity_gpu.py -x -q > $O/pytest_c4iter.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_c4iter.log
timeout 600 python bench.py --config c4 --steps 5 > $O/bench_c4.json 2>&1; echo "bench c4 rc=$?"; tail -c 700 $O/bench_c4.json; echo
timeout 300 python bench.py --config c3 --steps 5 > $O/bench_c3.json 2>&1; echo "bench c3 rc=$?"; python -c "import json;d=json.loads(open('$O/bench_c3.json').read().splitlines()[-1]);print(d['value'],d['ms_per_step'])"
[ "${SKIP_C5:-0}" = "1" ] || timeout 600 python bench.py --config c5 --steps 3 > $O/bench_c5.json 2>&1; echo "bench c5 rc=$?"; python -c "import json;d=json.loads(open('$O/bench_c5.json').read().splitlines()[-1]);print(d['value'],d['ms_per_step'])"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/kernels_c4_16384.csv timeout 600 python tools/prof_primitives.py --size 16384 --random 0.5 \
    --ops ccl,reach,maxvol --reps 2 > /dev/null 2>&1
echo "ncu c4 rc=$?"
python tools/launches.py $O/kernels_c4_16384.csv

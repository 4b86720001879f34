# quick A/B: C2 chain value + C4 kernels + parity subset
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_ccl_gpu.py tests/test_reach_gpu.py tests/test_executor_gpu.py -x -q > $O/pytest_ab.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_ab.log
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-primitives --alt-steps 0 > $O/bench_ab.json 2>&1; python -c "import json;d=json.loads(open('$O/bench_ab.json').read().splitlines()[-1]);print('C2', d['value'], d['ms_per_step'])"
timeout 600 python bench.py --config c4 --steps 5 > $O/bench_c4.json 2>&1; python -c "import json;d=json.loads(open('$O/bench_c4.json').read().splitlines()[-1]);print('C4', d['value'],d['ms_per_step'],d['config']['densities'])"
timeout 600 python bench.py --config c3 --steps 5 > $O/bench_c3.json 2>&1; python -c "import json;d=json.loads(open('$O/bench_c3.json').read().splitlines()[-1]);print('C3', d['value'],d['ms_per_step'])"
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_tile \
    --log-file $O/ab_k.csv timeout 600 python tools/prof_primitives.py --size 16384 --random 0.5 --ops ccl,reach --reps 2 > /dev/null 2>&1
python tools/launches.py $O/ab_k.csv

O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu.log
for c in c1 c3; do
timeout 300 python bench.py --config $c --steps 5 > $O/bench_$c.json 2>&1; python -c "import json;d=json.loads(open('$O/bench_$c.json').read().splitlines()[-1]);print('$c', d['value'],d['ms_per_step'], d['e2e'])"
done

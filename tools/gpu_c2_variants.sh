# C2 chain value for several variant builds (VS="a b c"), base first; then parity of the last
O=gpurun_out; mkdir -p $O
for v in base $VS; do
  lib=""; [ "$v" != base ] && lib=paper_2010_07284_b200/variants/$v.so
  SLCS_LIB_PATH=$lib timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-primitives --alt-steps 0 > $O/c2_$v.json 2>&1
  python -c "import json;d=json.loads(open('$O/c2_$v.json').read().splitlines()[-1]);print('$v C2', round(d['value'],1), round(d['ms_per_step'],3))"
done
for v in $VS; do
SLCS_LIB_PATH=paper_2010_07284_b200/variants/$v.so timeout 900 python -m pytest tests/test_reach_gpu.py tests/test_executor_gpu.py tests/test_acceptance_gpu.py -x -q 2>&1 | tail -1
done

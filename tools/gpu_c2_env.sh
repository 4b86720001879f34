# C2 chain value under env settings: ENVS="A=1 B=2;C=3" (';'-separated runs), base first
O=gpurun_out; mkdir -p $O
IFS=';' read -ra RUNS <<< "base;$ENVS"
for e in "${RUNS[@]}"; do
  [ "$e" = base ] && ev="" || ev="$e"
  env $ev timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-primitives --alt-steps 0 > $O/c2_env.json 2>&1
  python -c "import json;d=json.loads(open('$O/c2_env.json').read().splitlines()[-1]);print('[$e] C2', round(d['value'],1), round(d['ms_per_step'],3))"
done

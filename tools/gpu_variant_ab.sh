# A/B of a variant build (paper_2010_07284_b200/variants/$V.so) against the default build
O=gpurun_out; mkdir -p $O
for lib in "" "paper_2010_07284_b200/variants/$V.so"; do
  tag=${lib:+$V}; tag=${tag:-base}
  SLCS_LIB_PATH=$lib timeout 600 python bench.py --config c4 --steps 5 --no-e2e --no-cpu-baseline > $O/ab_c4_$tag.json 2>&1
  python -c "import json;d=json.loads(open('$O/ab_c4_$tag.json').read().splitlines()[-1]);print('$tag C4', round(d['ms_per_step'],3), {k:(round(v['ccl_ms'],3),round(v['reach_ms'],3)) for k,v in d['config']['densities'].items()})"
  if [ -n "$C2" ]; then SLCS_LIB_PATH=$lib timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-primitives --alt-steps 0 > $O/ab_c2_$tag.json 2>&1
  python -c "import json;d=json.loads(open('$O/ab_c2_$tag.json').read().splitlines()[-1]);print('$tag C2', d['value'], d['ms_per_step'])"; fi
  SLCS_LIB_PATH=$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_tile \
    --log-file $O/ab_k_$tag.csv timeout 600 python tools/prof_primitives.py --size 16384 --random 0.5 --ops ccl,reach,maxvol --reps 2 > /dev/null 2>&1
  python tools/launches.py $O/ab_k_$tag.csv
done

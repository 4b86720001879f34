# per-kernel ncu times (KRE regex) for the base build and variant builds VS="a b"
O=gpurun_out; mkdir -p $O
for v in base $VS; do
  lib=""; [ "$v" != base ] && lib=paper_2010_07284_b200/variants/$v.so
  SLCS_LIB_PATH=$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"$KRE" \
    --log-file $O/kv_$v.csv timeout 600 python tools/prof_primitives.py ${PARGS:---size 16384 --random 0.5 --ops ccl --reps 3} > /dev/null 2>&1
  echo "[$v]"; python tools/launches.py $O/kv_$v.csv | tail -n +2
done

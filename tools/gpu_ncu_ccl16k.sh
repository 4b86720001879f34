O=gpurun_out; mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:"k_tile_local|k_tile_merge|k_tile_labels|k_root_flatten" -c 5 -f -o $O/ccl16k \
    timeout 600 python tools/prof_primitives.py --reps 1 --size 16384 --random 0.5 --ops ccl > $O/ncu_ccl16k.log 2>&1; echo "ncu rc=$?"; tail -2 $O/ncu_ccl16k.log

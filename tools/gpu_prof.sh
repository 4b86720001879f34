#!/bin/bash
# primitive table at C4 size + ncu --set full captures of the top kernels
O=gpurun_out; mkdir -p $O
timeout 300 python tools/prim_table.py 16384 > $O/prim_16384.txt 2>&1; echo "prim rc=$?"; head -12 $O/prim_16384.txt
timeout 300 python tools/prim_table.py 4096 > $O/prim_4096.txt 2>&1; echo "prim4k rc=$?"; head -12 $O/prim_4096.txt
ncu --set full --clock-control none --import-source on -k regex:k_tile_local -s 1 -c 1 -f -o $O/tile_local_4096 \
    timeout 600 python tools/prof_primitives.py --reps 2 --ops reach > $O/ncu_full1.log 2>&1; echo "ncu1 rc=$?"; tail -3 $O/ncu_full1.log
ncu --set full --clock-control none --import-source on -k regex:k_tile_merge -s 1 -c 1 -f -o $O/tile_merge_4096 \
    timeout 600 python tools/prof_primitives.py --reps 2 --ops reach > $O/ncu_full2.log 2>&1; echo "ncu2 rc=$?"; tail -3 $O/ncu_full2.log
ncu --set full --clock-control none --import-source on -k regex:"k_near|k_threshold|k_tile_local|k_tile_labels|k_reach_select" -c 12 -f -o $O/prims_16384 \
    timeout 600 python tools/prof_primitives.py --reps 1 --size 16384 --random 0.5 --ops near,reach,ccl > $O/ncu_full3.log 2>&1; echo "ncu3 rc=$?"; tail -3 $O/ncu_full3.log
ls -la $O

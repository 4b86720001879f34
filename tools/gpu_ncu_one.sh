#!/bin/bash
# ncu --set full of one kernel: KRE (regex) from tools/prof_primitives.py $PARGS
O=gpurun_out; mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s ${SKIP:-1} -c 1 -f -o $O/$NAME \
    timeout 600 python tools/prof_primitives.py $PARGS > $O/ncu_$NAME.log 2>&1; echo "ncu rc=$?"; tail -2 $O/ncu_$NAME.log

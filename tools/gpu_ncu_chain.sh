#!/bin/bash
# ncu --set full of the config-2 chain's fused reach kernel (graph off, 8-step chain)
O=gpurun_out; mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:"k_reach_fused" -s 3 -c 1 -f -o $O/reach_fused_chain \
    timeout 600 python tools/chain_timing.py 4096 > $O/ncu_chain.log 2>&1; echo "ncu rc=$?"; tail -2 $O/ncu_chain.log

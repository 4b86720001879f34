#!/bin/bash
# Copy one tools/gpu_round2.sh result set from gpurun_out/ into profiles/ as r<tag>_*.
#   bash tools/save_profiles.sh 02d
set -e
t=$1; O=gpurun_out; P=profiles
tail -1 $O/bench.json > $P/r${t}_bench_c2.json
tail -1 $O/bench_ref.json > $P/r${t}_bench_c2_reference.json
python tools/launches.py $O/launches_bench.csv > $P/r${t}_launches_c2.txt
python tools/launches.py $O/launches_bench.csv --json $P/r${t}_launches_c2.json > /dev/null
cp $O/traffic_chain.json $P/r${t}_traffic_chain.json
cp $O/kernels_c4_16384.json $P/r${t}_kernels_c4_16384.json
python tools/ncu_summary.py $O/chain_full.ncu-rep > $P/r${t}_ncu_reach_chain_full.txt 2>&1 || true
python tools/ncu_lines.py $O/chain_full.ncu-rep k_reach_chain 30 >> $P/r${t}_ncu_reach_chain_full.txt 2>&1 || true
cp $O/pytest_gpu.log $P/r${t}_pytest_gpu.log
cp $O/smoke.log $P/r${t}_smoke.log
cp $O/chain_phases.txt $P/r${t}_chain_phases.txt
ls $P/r${t}_*

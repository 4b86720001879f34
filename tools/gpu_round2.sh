#!/bin/bash
# One gpurun call (round 2 evidence): GPU suite, smoke, the default bench line and
# the reference arm, ncu launch list of the bench, DRAM traffic of the headline
# kernel (k_reach_chain) and the C4 kernels, the chain's phase timeline and the
# grid-barrier microbenchmark.   gpurun --timeout 3000 -- 'bash tools/gpu_round2.sh'
mkdir -p gpurun_out
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/smi.txt 2>&1
nproc > $O/nproc.txt
if [ "${SKIP_TESTS:-0}" = "0" ]; then
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 180 python __graft_entry__.py > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
fi
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -c 300 $O/bench.json; tail -3 $O/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2>&1; echo "ref rc=$?"; tail -c 300 $O/bench_ref.json
SLCS_PHASE_TIMING=1 timeout 120 python tools/prof_chain.py 1000 3 2> $O/chain_phases.txt > /dev/null; tail -1 $O/chain_phases.txt
[ -x tools/ubench_barrier ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_barrier tools/ubench_barrier.cu
timeout 60 ./tools/ubench_barrier > $O/ubench_barrier.txt 2>&1; tail -3 $O/ubench_barrier.txt
if [ "${SKIP_NCU:-0}" = "0" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_bench.csv \
    timeout 900 python bench.py --steps 1 --warmup 3 --alt-steps 0 --no-cpu-baseline --no-e2e --no-primitives --no-extra > $O/ncu_bench.log 2>&1
echo "ncu launches rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/traffic_chain.csv timeout 600 python tools/prof_chain.py 1000 2 > /dev/null 2>&1
echo "ncu traffic rc=$?"
python tools/launches.py $O/launches_bench.csv $O/traffic_chain.csv --json $O/traffic_chain.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/kernels_c4_16384.csv timeout 600 python tools/prof_primitives.py --size 16384 --random 0.5 \
    --ops ccl,reach,maxvol --reps 2 > /dev/null 2>&1
echo "ncu c4 rc=$?"
python tools/launches.py $O/kernels_c4_16384.csv --json $O/kernels_c4_16384.json
ncu --set full --import-source on --clock-control none -k regex:k_reach_chain -c 1 -o $O/chain_full -f \
    timeout 600 python tools/prof_chain.py 1000 1 > /dev/null 2>&1
echo "ncu full rc=$?"
fi

#!/bin/bash
# One gpurun call: parity tests, smoke, headline bench + reference arm, the other
# configs, ncu launch list of the bench command and per-launch DRAM traffic.
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh'
mkdir -p gpurun_out
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/smi.txt 2>&1
nproc > $O/nproc.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 180 python __graft_entry__.py > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -c 600 $O/bench.json; tail -3 $O/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2>&1; echo "ref rc=$?"; tail -c 300 $O/bench_ref.json
for c in c1 c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps 5 > $O/bench_$c.json 2>&1; echo "bench $c rc=$?"; tail -c 400 $O/bench_$c.json; echo
done
if [ "${SKIP_NCU:-0}" = "0" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_bench.csv \
    timeout 900 python bench.py --steps 1 --warmup 3 --alt-steps 0 --no-cpu-baseline --no-e2e --no-primitives > $O/ncu_bench.log 2>&1
echo "ncu launches rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/traffic_4096.csv timeout 600 python tools/prof_primitives.py --reps 2 --ops reach,near,threshold > /dev/null 2>&1
echo "ncu traffic rc=$?"
python tools/launches.py $O/launches_bench.csv $O/traffic_4096.csv
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/kernels_c4_16384.csv timeout 600 python tools/prof_primitives.py --size 16384 --random 0.5 \
    --ops ccl,reach,maxvol --reps 2 > /dev/null 2>&1
echo "ncu c4 rc=$?"
python tools/launches.py $O/kernels_c4_16384.csv
fi

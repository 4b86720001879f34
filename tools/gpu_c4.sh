O=gpurun_out; mkdir -p $O
timeout 600 python bench.py --config c4 --steps 5 > $O/bench_c4.json 2>&1; echo "rc=$?"; tail -c 1500 $O/bench_c4.json

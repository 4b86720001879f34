O=gpurun_out; mkdir -p $O
for part in X H V; do
SLCS_MERGE_PART=$part ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_tile_merge \
    --log-file $O/merge_$part.csv timeout 600 python tools/prof_primitives.py --size 16384 --random 0.5 --ops ccl --reps 2 > /dev/null 2>&1
echo "part $part"; python tools/launches.py $O/merge_$part.csv
done

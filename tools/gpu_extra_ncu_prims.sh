ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/prim16k_ncu.csv timeout 300 python tools/prim_table.py 16384 > /dev/null 2>&1
python tools/launches.py gpurun_out/prim16k_ncu.csv

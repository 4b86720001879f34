#!/bin/bash
# quick loop: GPU parity tests + primitive tables (+ optional extra command in $EXTRA)
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest_gpu.log
timeout 300 python tools/prim_table.py 16384 > $O/prim_16384.txt 2>&1; echo "prim rc=$?"; head -13 $O/prim_16384.txt
timeout 300 python tools/prim_table.py ${PRIM2:-65536} > $O/prim_2.txt 2>&1; echo "prim2 rc=$?"; head -13 $O/prim_2.txt
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi

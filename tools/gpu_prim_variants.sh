# primitive table rows (OPS regex) at size N for base and variants VS
O=gpurun_out; mkdir -p $O
for v in base $VS; do
  lib=""; [ "$v" != base ] && lib=paper_2010_07284_b200/variants/$v.so
  echo "[$v]"; SLCS_LIB_PATH=$lib timeout 600 python tools/prim_table.py ${N:-16384} 2>&1 | grep -E "${OPS:-near}" | grep -v "^{"
done

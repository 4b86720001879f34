# Primitive table (bench.py's primitives_c4 at SIZE, default 16384) for the base
# build and each variant .so in VS; OPS = a regex of the rows to print.
for v in base $VS; do
  lib=""; [ "$v" != base ] && lib=paper_2010_07284_b200/variants/$v.so
  echo "== $v"; SLCS_LIB_PATH=$lib python tools/prim_table.py ${SIZE:-16384} 2>&1 | grep -E "^(${OPS:-ccl|reach|maxvol}) "
done

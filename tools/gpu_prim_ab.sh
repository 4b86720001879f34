for v in base $VS; do
  lib=""; [ "$v" != base ] && lib=paper_2010_07284_b200/variants/$v.so
  echo "== $v"; SLCS_LIB_PATH=$lib python tools/prim_table.py 16384 2>&1 | grep -E "^(ccl|reach|maxvol) "
done

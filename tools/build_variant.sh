#!/bin/bash
# Build libslcs with extra nvcc flags into paper_2010_07284_b200/variants/<name>.so
# (A/B measurements: SLCS_LIB_PATH=<that .so> python ...).
#   bash tools/build_variant.sh v3 -DSLCS_TL_MINB=3
set -e
name=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
D=$R/paper_2010_07284_b200/variants/$name; mkdir -p $D
objs=()
for f in $R/paper_2010_07284_b200/csrc/*.cu; do
  o=$D/$(basename $f).o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 \
       --expt-relaxed-constexpr "$@" -c $f -o $o &
  objs+=($o)
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D.so "${objs[@]}" -cudart shared -lcuda -lz \
     -Xlinker -rpath,/usr/local/cuda/lib64
echo $D.so

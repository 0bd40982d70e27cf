#!/bin/bash
# Debug variant of libsetbwte.so with device bounds checks (SB_DEBUG) in every
# source -> build/variants/dbg/libsetbwte.so; run tests with
#   SETBWTE_LIB=build/variants/dbg/libsetbwte.so python -m pytest tests -m gpu
set -e
cd "$(dirname "$0")/.."
d=build/variants/dbg; mkdir -p $d
objs=""
for f in paper_1410_0562_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Iinclude -Ipaper_1410_0562_b200/csrc -DSB_DEBUG -c $f -o $d/$b.o &
  objs="$objs $d/$b.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $d/libsetbwte.so $objs
echo $d/libsetbwte.so

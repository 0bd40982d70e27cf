#!/bin/bash
# Build an experimental variant of libsetbwte.so with extra nvcc flags for one
# source file:  tools/variant.sh <name> <file.cu> "-DFOO=1 ..."
#   -> build/variants/<name>/libsetbwte.so  (use with SETBWTE_LIB=...)
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; flags=$3
python -c "from paper_1410_0562_b200 import _build; _build.build()" >/dev/null
d=build/variants/$name; mkdir -p $d
objs=""
for f in paper_1410_0562_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  if [ "$b.cu" = "$src" ]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      -Iinclude -Ipaper_1410_0562_b200/csrc $flags -Xptxas -v -c $f -o $d/$b.o > $d/$b.ptxas.log 2>&1
    objs="$objs $d/$b.o"
  else
    objs="$objs build/$b.o"
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $d/libsetbwte.so $objs
echo $d/libsetbwte.so

#!/bin/bash
# ncu --set full captures of selected kernels of one c3 build (20M x 100 bp,
# M = 2^27; run on the GPU box):  bash tools/prof_c3.sh <out-name> "<regex>:<skip>" ...
out=$1; shift
args="--reads 20000000 --M 134217728 $C3_ARGS"
python tools/run_once.py $args > gpurun_out/${out}_plain.log 2>&1 || { echo plain run failed; exit 1; }
i=0
for spec in "$@"; do
  re=${spec%%:*}; sk=${spec##*:}
  ncu --set full --clock-control none --import-source on -k regex:"$re" -s $sk -c 1 \
      -o gpurun_out/${out}_$i python tools/run_once.py $args > gpurun_out/${out}_ncu_$i.log 2>&1
  echo "ncu $re skip=$sk rc=$?"
  i=$((i+1))
done

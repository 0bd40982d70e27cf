#!/bin/bash
# ncu --set full captures of selected kernels of one c2 build (run on the GPU box)
# usage: tools/prof.sh <out-name> "<regex1>:<skip1>" "<regex2>:<skip2>" ...
out=$1; shift
python tools/run_once.py > gpurun_out/plain.log 2>&1 || { echo plain run failed; exit 1; }
i=0
for spec in "$@"; do
  re=${spec%%:*}; sk=${spec##*:}
  ncu --set full --clock-control none --import-source on -k regex:"$re" -s $sk -c 1 \
      -o gpurun_out/${out}_$i python tools/run_once.py > gpurun_out/ncu_$i.log 2>&1
  echo "ncu $re skip=$sk rc=$?"
  i=$((i+1))
done

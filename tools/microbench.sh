#!/bin/bash
# Roofline microbenchmarks on the GPU box:
#   bash tools/microbench.sh r01   -> gpurun_out/microbench.json (copy to profiles/<round>_microbench.json)
set -e
cd "$(dirname "$0")/.."
mkdir -p build gpurun_out
[ -x build/microbench ] || nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/microbench tools/microbench.cu
./build/microbench > gpurun_out/microbench.json
cat gpurun_out/microbench.json

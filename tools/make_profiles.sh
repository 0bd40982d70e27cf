#!/bin/bash
# Round profile artefacts (run on the GPU box):  bash tools/make_profiles.sh r01
r=${1:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/${r}_gpu.txt
python bench.py > gpurun_out/${r}_bench.json 2> gpurun_out/${r}_bench.err; echo bench_rc=$?
python bench.py --impl reference > gpurun_out/${r}_ref.json 2> gpurun_out/${r}_ref.err; echo ref_rc=$?
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${r}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/${r}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${r}_ncu_launches.log 2>&1; echo launches_rc=$?
bash tools/prof.sh ${r}_full "digit_scatter:0" "bitonic_kernel:0" "compute_ranks:4" "gather_kernel:5" \
    "insert_kernel:5" "digit_hist:0" "tiny_kernel:0"

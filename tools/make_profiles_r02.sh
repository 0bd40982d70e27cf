#!/bin/bash
# Round-2 profile artefacts on the GPU box (c3 = the metric's config):
#   bash tools/make_profiles_r02.sh   -> gpurun_out/r02_*
r=r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/${r}_gpu.txt
python bench.py > gpurun_out/${r}_bench.json 2> gpurun_out/${r}_bench.err; echo bench_rc=$?
python bench.py --workload c2 > gpurun_out/${r}_bench_c2.json 2> gpurun_out/${r}_bench_c2.err; echo c2_rc=$?
python bench.py --impl reference > gpurun_out/${r}_ref.json 2> gpurun_out/${r}_ref.err; echo ref_rc=$?
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${r}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv \
    --log-file gpurun_out/${r}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${r}_ncu_launches.log 2>&1; echo launches_rc=$?
bash tools/prof_c3.sh ${r}_full "local_digit:1" "gather_kernel:8" "compute_ranks:8" \
    "digit_scatter:1" "insert_kernel:10" "digit_hist:1" "pack_kernel:5"

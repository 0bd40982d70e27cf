#!/bin/bash
# serialised per-kernel times of one c3 build (ncu launch list) -> gpurun_out/c3_launches_$1.csv
tag=${1:-x}
python tools/run_once.py --reads 20000000 --M 134217728 > /dev/null 2>&1 || { echo c3 run failed; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches_$tag.csv \
    python tools/run_once.py --reads 20000000 --M 134217728 > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/c3_launches_$tag.csv | head -12

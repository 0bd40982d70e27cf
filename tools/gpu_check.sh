#!/bin/bash
# one gpurun call: gpu tests (fast subset) + bench line
tag=${1:-x}
timeout 600 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -4 gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench_rc=$?
python - <<PY
import json
d=json.load(open('gpurun_out/bench_$tag.json'))
print('value', d['value'], 'ms/step', d['ms_per_step'], 'e2e', d['e2e']['value'])
print('kernels', d['kernel_ms_per_step'])
print('roofline', d['roofline']['kernel'], d['roofline']['frac'])
PY
tail -2 gpurun_out/bench_$tag.err
# serialized per-kernel times of one c2 build (ncu launch list)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv python tools/run_once.py > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/launches_$tag.csv | head -30

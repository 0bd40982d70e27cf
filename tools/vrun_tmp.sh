for o in "sort_lanes=0" "sort_lanes=1" "sort_lanes=2"; do
  python bench.py --no-cpu-baseline --steps 20 --warmup 3 --option $o > gpurun_out/var.json 2> gpurun_out/var.err
  python -c "import json; d=json.load(open('gpurun_out/var.json')); print('$o', d['value'], d['ms_per_step'])"
done

timeout 900 python -m pytest tests -m "gpu" -x -q 2>&1 | tail -1
for v in head cur head cur; do
  if [ $v = cur ]; then L=""; else L=build/variants/head/libsetbwte.so; fi
  SETBWTE_LIB=$L python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/var.json 2> gpurun_out/var.err
  python -c "import json; d=json.load(open('gpurun_out/var.json')); print('$v', d['value'], d['e2e']['value'], d['ms_per_step'], d['parity_vs_oracle'])"
done
pids=""
for i in $(seq 1 $(nproc)); do python -c "while True: pass" & pids="$pids $!"; done
sleep 1
for v in head cur; do
  if [ $v = cur ]; then L=""; else L=build/variants/head/libsetbwte.so; fi
  SETBWTE_LIB=$L python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/var.json 2> gpurun_out/var.err
  python -c "import json; d=json.load(open('gpurun_out/var.json')); print('loaded $v', d['value'], d['e2e']['value'], d['ms_per_step'])"
done
kill $pids

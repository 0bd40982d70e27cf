#!/bin/bash
# A/B a variant library against the in-tree one on the GPU box:
#   tools/ab.sh <variant.so> [rounds] [bench args...]  -> value / e2e / frac per run
v=$1; r=${2:-3}; shift 2
for i in $(seq $r); do
  for lib in "" "$v"; do
    SETBWTE_LIB=$lib python bench.py --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('${lib:-base}', d['value'], d['e2e']['value'], d['roofline']['frac'], d['ms_per_step'])"
  done
done

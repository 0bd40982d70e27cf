#!/bin/bash
# A/B library options on the GPU box, alternating runs:
#   tools/ab_opt.sh <rounds> "<optsA>" "<optsB>" [bench args...]
#   opts: space-separated key=value (empty string = defaults)
r=$1; a=$2; b=$3; shift 3
for i in $(seq $r); do
  for o in "$a" "$b"; do
    args=""
    for kv in $o; do args="$args --option $kv"; done
    python bench.py --no-cpu-baseline $args "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('[${o:-default}]', d['value'], 'e2e', d['e2e']['value'], 'ms', d['ms_per_step'], 'frac', d['roofline']['frac'], {k: round(v,2) for k,v in d['stage_ms_per_step'].items()})"
  done
done

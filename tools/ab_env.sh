#!/bin/bash
# A/B an environment setting: tools/ab_env.sh <rounds> "<envA>" "<envB>" [bench args...]
r=$1; a=$2; b=$3; shift 3
for i in $(seq $r); do
  for e in "$a" "$b"; do
    env $e python bench.py --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('[${e}]', d['value'], 'e2e', d['e2e']['value'], 'ms', d['ms_per_step'], {k: round(v,2) for k,v in d['stage_ms_per_step'].items()})"
  done
done

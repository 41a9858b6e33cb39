#!/bin/bash
# A/B of environment settings: bench step / stage times for each "VAR=value" given, alternating twice.
for i in 1 2; do
  for e in "$@"; do
    env $e timeout 300 python bench.py --steps 20 --warmup 5 --no-cfg3 --no-cudnn --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages_ms']
print('$e'.ljust(28), round(d['ms_per_step'],4), ' '.join(f'{k.replace(\"scfa_\",\"\")}={v}' for k,v in s.items()))"
  done
done

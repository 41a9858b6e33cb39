#!/bin/bash
# A/B of whole trees (each with its own built library): "dir[:ENV=val,...]" relative to the repo root.
for i in 1 2; do
  for spec in "$@"; do
    d=${spec%%:*}; envs=""; [ "$spec" != "$d" ] && envs=$(echo ${spec#*:} | tr ',' ' ')
    (cd "$GRAFT_REPO_ROOT/$d" && env $envs timeout 300 python bench.py --steps 20 --warmup 5 --no-cfg3 --no-cudnn --no-cpu-baseline 2>/dev/null) | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages_ms']
print('$spec'.ljust(28), round(d['ms_per_step'],4), ' '.join(f'{k.replace(\"scfa_\",\"\")}={v}' for k,v in s.items()))"
  done
done

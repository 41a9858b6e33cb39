#!/bin/bash
# A/B of environment settings on the full bench line (cfg2 step, cfg3 QK, hash T=16k, dense),
# each "VAR=value" given, alternating twice.
for i in 1 2; do
  for e in "$@"; do
    env $e timeout 400 python bench.py --steps 10 --warmup 3 --no-cudnn --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages_ms']
print('$e'.ljust(22), 'cfg2', round(d['ms_per_step'],4), 'cfg3', round(d['cfg3_qk']['ms_per_step'],3), 't16k', round(d['hash_t16k']['ms_per_step'],3), 'dense', round(d['dense_causal']['ms_per_step'],3), ' '.join(f'{k.replace(\"scfa_\",\"\")}={v}' for k,v in s.items() if 'attn' not in k))"
  done
done

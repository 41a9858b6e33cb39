#!/bin/bash
# A/B of alternative builds on the full bench line (cfg2 step, cfg3 QK, hash T=16k, dense):
# library paths relative to the repo root ("tree" = the in-tree build), alternating twice.
for i in 1 2; do
  for lib in "$@"; do
    if [ "$lib" = tree ]; then L=""; else L="$GRAFT_REPO_ROOT/$lib"; fi
    SCFA_LIB=$L timeout 400 python bench.py --steps 10 --warmup 3 --no-cudnn --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages_ms']
print('$lib'.ljust(22), 'cfg2', round(d['ms_per_step'],4), 'cfg3', round(d['cfg3_qk']['ms_per_step'],3), 't16k', round(d['hash_t16k']['ms_per_step'],3), 'dense', round(d['dense_causal']['ms_per_step'],3), ' '.join(f'{k.replace(\"scfa_attn_\",\"\")}={v}' for k,v in s.items() if 'attn' in k))"
  done
done

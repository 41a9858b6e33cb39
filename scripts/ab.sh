#!/bin/bash
# A/B: bench stage times of the in-tree build vs ab/libscfa_head.so, alternating.
for i in 1 2; do
  for lib in "" "ab/libscfa_head.so"; do
    SCFA_LIB=${lib:+$GRAFT_REPO_ROOT/$lib} timeout 300 python bench.py --steps 20 --warmup 5 --no-cfg3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages_ms']
print('${lib:-tree}'.ljust(22), round(d['ms_per_step'],4), 'fwd', s['scfa_attn_fwd'], 'dq', s['scfa_attn_bwd_dq'], 'dkdv', s['scfa_attn_bwd_dkdv'], 'dense', round(d['dense_causal']['ms_per_step'],3))"
  done
done

#!/bin/bash
# A/B of a Python-side flag: bench stage times with paper_2306_01160_b200.hash_sparse.$1 on / off.
for i in 1 2; do
  for val in True False; do
    timeout 300 python -c "
import sys, runpy
import paper_2306_01160_b200.hash_sparse as h
setattr(h, '$1', $val)
sys.argv = ['bench.py', '--steps', '20', '--warmup', '5', '--no-cfg3']
runpy.run_path('bench.py', run_name='__main__')" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stages_ms']
print('$1=$val'.ljust(26), round(d['ms_per_step'],4), 'fwd', s['scfa_attn_fwd'], 'dq', s['scfa_attn_bwd_dq'], 'dkdv', s['scfa_attn_bwd_dkdv'], 'e2e', round(d['e2e']['ms_per_step'],3))"
  done
done

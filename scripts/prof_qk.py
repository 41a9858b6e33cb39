"""One cfg3 QK-sparse fwd+bwd step (B=4 H=12 T=16384 D=64, drop 0.5), repeated: a short
command to run under ncu (needs a GPU).    python scripts/prof_qk.py [steps] [drop]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_2306_01160_b200 as scfa

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
drop = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
B, H, T, D = 4, 12, 16384, 64
g = torch.Generator(device="cuda").manual_seed(16)
q, k, v, dO = (torch.randn((B, T, H, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
qk = torch.from_numpy(scfa.random_keep(B, T, H, drop, 6)).cuda()
kk = torch.from_numpy(scfa.random_keep(B, T, H, drop, 7)).cuda()
for _ in range(steps):
    scfa.qk_sparse_attention_fwd_bwd(q, k, v, qk, kk, dO, check=False)
torch.cuda.synchronize()
print("done", steps, "QK steps at drop", drop)

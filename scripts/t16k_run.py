"""One hash fwd+bwd at the north-star shape (B=4 H=12 T=16384 D=64, 16 buckets) for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_01160_b200 import hash_sparse as hs  # noqa: E402

B, H, T, D, nb = 4, 12, 16384, 64, 16
g = torch.Generator(device="cuda").manual_seed(17)
q, k, v, dO = (torch.randn((B, T, H, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
ids = torch.randint(0, nb, (B, T, H), device="cuda", generator=g)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    hs._fwd_bwd(q, k, v, ids, ids, dO)
torch.cuda.synchronize()

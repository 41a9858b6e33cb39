"""Kernel breakdown of one hash fwd+bwd at D = 64 and 128 (B=2, T=16384, nb=16; diagnostics)."""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_01160_b200 import hash_sparse as hs  # noqa: E402

for D in (64, 128):
    B, T, H, nb = 2, 16384, 12, 16
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v, dO = (torch.randn((B, T, H, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    ids = torch.randint(0, nb, (B, T, H), device="cuda", generator=g)
    for _ in range(3):
        hs._fwd_bwd(q, k, v, ids, ids, dO)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        hs._fwd_bwd(q, k, v, ids, ids, dO)
        torch.cuda.synchronize()
    print("D =", D)
    for e in sorted(prof.key_averages(), key=lambda e: -e.device_time_total)[:6]:
        print(f"   {e.key[:60]:60s} {e.device_time_total:9.1f} us")

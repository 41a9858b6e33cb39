"""Kernel breakdown of one cfg3 QK-sparse fwd+bwd call (torch.profiler; diagnostics)."""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_01160_b200 as scfa  # noqa: E402

B, H, T, D, drop = 4, 12, 16384, 64, 0.5
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(16)
q, k, v, dO = (torch.randn((B, T, H, D), device=dev, generator=g).to(torch.bfloat16) for _ in range(4))
qk = torch.from_numpy(scfa.random_keep(B, T, H, drop, 6)).to(dev)
kk = torch.from_numpy(scfa.random_keep(B, T, H, drop, 7)).to(dev)
f = lambda: scfa.qk_sparse_attention_fwd_bwd(q, k, v, qk, kk, dO)
for _ in range(3):
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    f()
e1.record()
torch.cuda.synchronize()
print("eager ms/call", e0.elapsed_time(e1) / 10)
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    f()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=18, max_name_column_width=48))

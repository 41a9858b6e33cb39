"""Hash fwd+bwd at D=128 (B=4 H=12 T=8192 nb=16), CUDA-graph replay, ms per step (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2306_01160_b200 as scfa
from paper_2306_01160_b200 import hash_sparse as hs

B, T, H, D = 4, 8192, 12, 128
g = torch.Generator(device="cuda").manual_seed(0)
x = [torch.randn((B, T, H, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(4)]
h = torch.randint(0, 16, (B, T, H), device="cuda", generator=g)
f = lambda: hs._fwd_bwd(x[0], x[1], x[2], h, h, x[3], exclude_self=True)
for _ in range(3):
    f()
torch.cuda.synchronize()
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    f()
torch.cuda.current_stream().wait_stream(s)
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr):
    f()
gr.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    gr.replay()
e1.record(); torch.cuda.synchronize()
print(f"D=128 hash fwd+bwd: {e0.elapsed_time(e1) / 20:.4f} ms")

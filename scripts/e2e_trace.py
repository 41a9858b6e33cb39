"""GPU timeline of the public host-buffer fwd+bwd call (diagnostics, needs a GPU): the
per-slice upload / compute / download marks recorded by hash_sparse._fwd_bwd_host."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2306_01160_b200 as scfa
from paper_2306_01160_b200 import hash_sparse as hs

B, T, H, D = 4, 8192, 12, 64
x = [torch.randn((B, T, H, D)).to(torch.bfloat16).pin_memory() for _ in range(4)]
h = torch.randint(0, 16, (B, T, H)).pin_memory()
outs = [torch.empty((B, T, H, D), dtype=torch.bfloat16, pin_memory=True)] + [
    torch.empty((B, T, H, D), dtype=torch.float32, pin_memory=True) for _ in range(3)]
for _ in range(3):
    scfa.hash_sparse_attention_fwd_bwd(x[0], x[1], x[2], h, h, x[3], out=outs)
torch.cuda.synchronize()
for rep in range(3):
    hs._TRACE = []
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e0.record()
    scfa.hash_sparse_attention_fwd_bwd(x[0], x[1], x[2], h, h, x[3], out=outs)
    e1 = torch.cuda.Event(enable_timing=True); e1.record()
    torch.cuda.synchronize()
    wall = 1e3 * (time.perf_counter() - t0)
    print(f"public call: {wall:.2f} ms wall, {e0.elapsed_time(e1):.2f} ms events")
    print("  ".join(f"{n}={e0.elapsed_time(e):.2f}" for n, e in hs._TRACE))
hs._TRACE = None

"""Time the host-input fwd+bwd path phases (diagnostics, needs a GPU)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2306_01160_b200 as scfa

B, T, H, D = 4, 8192, 12, 64
x = [torch.randn((B, T, H, D)).to(torch.bfloat16).pin_memory() for _ in range(4)]
h = torch.randint(0, 16, (B, T, H)).pin_memory()
outs = [torch.empty((B, T, H, D), dtype=torch.bfloat16, pin_memory=True)] + [torch.empty((B, T, H, D), dtype=torch.float32, pin_memory=True) for _ in range(3)]
for _ in range(2):
    scfa.hash_sparse_attention_fwd_bwd(x[0], x[1], x[2], h, h, x[3], out=outs)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    scfa.hash_sparse_attention_fwd_bwd(x[0], x[1], x[2], h, h, x[3], out=outs)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"host path: enqueue {1e3*(t1-t0):.1f} ms, total {1e3*(t2-t0):.1f} ms")
d = [t.cuda() for t in x]
hd = h.cuda()
torch.cuda.synchronize()
t0 = time.perf_counter()
for b in range(B):
    r = scfa.hash_sparse_attention_fwd_bwd(d[0][b:b+1], d[1][b:b+1], d[2][b:b+1], hd[b:b+1], hd[b:b+1], d[3][b:b+1])
torch.cuda.synchronize()
print(f"device chunks: {1e3*(time.perf_counter()-t0):.1f} ms")
t0 = time.perf_counter()
for t, o in zip(x, outs):
    o.copy_(t.cuda(non_blocking=True), non_blocking=True) if o.dtype == t.dtype else None
torch.cuda.synchronize()
print(f"copies alone (bf16 in/out): {1e3*(time.perf_counter()-t0):.1f} ms")
# phase-by-phase enqueue timing of the host path
from paper_2306_01160_b200 import hash_sparse as hs
dev = torch.device("cuda")
comp = torch.cuda.current_stream()
h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
for rep in range(2):
    tt = {}
    def tick(name, t0):
        tt[name] = tt.get(name, 0) + time.perf_counter() - t0
    for b in range(B):
        sl = slice(b, b + 1)
        t0 = time.perf_counter()
        with torch.cuda.stream(h2d):
            xs = [t[sl].to(dev, non_blocking=True) for t in (x[0], x[1], x[2], x[3], h)]
            ready = torch.cuda.Event(); ready.record(h2d)
        tick("h2d", t0); t0 = time.perf_counter()
        comp.wait_event(ready)
        for t in xs: t.record_stream(comp)
        outputs, dq, dk, dv, _ = hs._fwd_bwd(xs[0], xs[1], xs[2], xs[4], xs[4], xs[3])
        tick("compute", t0); t0 = time.perf_counter()
        done = torch.cuda.Event(); done.record(comp)
        with torch.cuda.stream(d2h):
            d2h.wait_event(done)
            for dst, src in zip(outs, (outputs.O, dq, dk, dv)):
                dst[sl].copy_(src, non_blocking=True)
                src.record_stream(d2h)
        tick("d2h", t0)
    t0 = time.perf_counter(); torch.cuda.synchronize(); tick("sync", t0)
    print({k: round(v * 1e3, 2) for k, v in tt.items()})

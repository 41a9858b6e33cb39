"""GPU timeline of the host-buffer fwd+bwd (diagnostics, needs a GPU): CUDA events on each
stream around each batch element's H2D, compute and D2H, relative to one start event."""
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
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e0.record()
    scfa.hash_sparse_attention_fwd_bwd(x[0], x[1], x[2], h, h, x[3], out=outs)
    e1 = torch.cuda.Event(enable_timing=True); e1.record()
    torch.cuda.synchronize()
    print(f"public call: {1e3 * (time.perf_counter() - t0):.2f} ms wall, {e0.elapsed_time(e1):.2f} ms events")

dev = torch.device("cuda")
comp = torch.cuda.current_stream()
h2d, d2h, _ = hs._copy_streams(dev)
for rep in range(2):
    ev = []
    def mark(name, s):
        e = torch.cuda.Event(enable_timing=True); e.record(s); ev.append((name, e))
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True); t_start.record(comp)
    h2d.wait_stream(comp); d2h.wait_stream(comp)
    host_t = {}
    for b in range(B):
        sl = slice(b, b + 1)
        t0 = time.perf_counter()
        with torch.cuda.stream(h2d):
            mark(f"h2d{b}-start", h2d)
            xs = [t[sl].to(dev, non_blocking=True) for t in (x[0], x[1], x[2], x[3], h)]
            mark(f"h2d{b}-end", h2d)
            ready = torch.cuda.Event(); ready.record(h2d)
        comp.wait_event(ready)
        for t in xs: t.record_stream(comp)
        mark(f"cmp{b}-start", comp)
        outputs, dq, dk, dv, _ = hs._fwd_bwd(xs[0], xs[1], xs[2], xs[4], xs[4], xs[3])
        mark(f"cmp{b}-end", comp)
        done = torch.cuda.Event(); done.record(comp)
        with torch.cuda.stream(d2h):
            d2h.wait_event(done)
            mark(f"d2h{b}-start", d2h)
            for dst, src in zip(outs, (outputs.O, dq, dk, dv)):
                dst[sl].copy_(src, non_blocking=True)
                src.record_stream(d2h)
            mark(f"d2h{b}-end", d2h)
        host_t[b] = 1e3 * (time.perf_counter() - t0)
    comp.wait_stream(d2h)
    mark("end", comp)
    torch.cuda.synchronize()
    print("host enqueue ms per element:", {k: round(v, 2) for k, v in host_t.items()})
    print("  ".join(f"{n}={t_start.elapsed_time(e):.2f}" for n, e in ev))

"""cfg2 K/V permute alone vs under the concurrent finish / tile-list kernels (diagnostics)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_2306_01160_b200 import hash_sparse as hs

B, T, H, D = 4, 8192, 12, 64
dev = torch.device("cuda")
k, v = (torch.randn((B, T, H, D), device=dev).to(torch.bfloat16) for _ in range(2))
ids = torch.randint(0, 16, (B, T, H), device=dev)
err = torch.zeros(1, dtype=torch.int32, device=dev)
hv, sb_, st_, sh_ = hs._hash_view(ids, B, H, T, "bth")
perm, rank, prob = hs._prepare_shared(hv, sb_, st_, sh_, B, H, T, D, err, True)
torch.cuda.synchronize()

def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay(); torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3

print(f"permute K,V alone: {timeit(lambda: hs._permute3([k, v], [rank, rank], T)):.1f} us")
def sched():
    p = hs.Problem(B, H, T, T, D, prob.q_idx, prob.k_idx, prob.q_hash, prob.k_hash, flags=prob.flags)
    p.set_runs(prob._lists["q_runs"] if "q_runs" in prob._lists else None, None) if False else None
    p.schedule("fwd", "dq", "dkdv")
print(f"schedule alone: {timeit(sched):.1f} us")
def both():
    main = torch.cuda.current_stream()
    side = hs._copy_streams(dev)[2]
    side.wait_stream(main)
    with torch.cuda.stream(side):
        hs._permute3([k, v], [rank, rank], T)
    sched()
    main.wait_stream(side)
print(f"permute || schedule: {timeit(both):.1f} us")

import os, sys, torch
sys.path.insert(0, "/root/repo")
from torch.profiler import profile, ProfilerActivity
from paper_2306_01160_b200 import hash_sparse as hs
for (B, T) in ((4, 8192), (2, 16384), (8, 4096)):
    H, D, nb = 12, 64, 16
    ids = torch.randint(0, nb, (B, T, H), device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    f = lambda: hs._prepare_shared(*hs._hash_view(ids, B, H, T, "bth"), B, H, T, D, err, True)
    for _ in range(5): f()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(10): f()
        torch.cuda.synchronize()
    for e in prof.key_averages():
        if "sort" in e.key:
            print(B, T, e.key[:40], round(e.device_time_total / e.count, 2), "us")

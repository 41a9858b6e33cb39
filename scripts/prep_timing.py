"""Time the index-preparation entry points alone at cfg2 shape (diagnostics, needs a GPU)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2306_01160_b200 import hash_sparse as hs

B, T, H, D = 4, 8192, 12, 64
dev = torch.device("cuda")


def timeit(fn, n=20):
    """CUDA-graph replay timing (host launch overhead excluded)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.current_stream().wait_stream(side)
    with torch.cuda.graph(g):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay()
    torch.cuda.synchronize()
    s.record()
    for _ in range(n):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3


def timeit_eager(fn, n=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3


x = torch.randn((B, T, H, D), device=dev).to(torch.bfloat16)
for nb in (1, 16, 300):
    h = torch.randint(0, nb, (B, T, H), device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    us = timeit(lambda: hs._prepare_shared(h, h.stride(0), h.stride(1), h.stride(2), B, H, T, D, err, True))
    h32 = h.to(torch.int32)
    us32 = timeit(lambda: hs._prepare_shared(h32, h32.stride(0), h32.stride(1), h32.stride(2), B, H, T, D, err, True))
    print(f"hash_prepare nb={nb}: int64 ids {us:.1f} us, int32 ids {us32:.1f} us")
perm, rank, prob = hs._prepare_shared(h, h.stride(0), h.stride(1), h.stride(2), B, H, T, D, err, True)
print(f"gather3: {timeit(lambda: hs._gather3([x, x, x], [perm, perm, perm], 'bthd')):.1f} us")
from paper_2306_01160_b200 import _lib
outs = [torch.empty((B, H, T, D), dtype=x.dtype, device=dev) for _ in range(3)]
strides = [x.stride(0), x.stride(1), x.stride(2)] * 3
def perm3():
    _lib.call("scfa_permute_rows3", 3, _lib.ptr_array([x, x, x]), _lib.ptr_array(outs), _lib.ptr_array([rank] * 3),
              _lib.i64_array(strides), 2, B, T, H, D, _lib.i64_array([T] * 3), _lib.stream_ptr())
print(f"permute3 (source order): {timeit(perm3):.1f} us")
g3 = hs._gather3([x, x, x], [perm, perm, perm], 'bthd')
perm3(); torch.cuda.synchronize()
print("permute3 == gather3:", all(torch.equal(a, b) for a, b in zip(g3, outs)))
print(f"gather1: {timeit(lambda: hs._gather3([x], [perm], 'bthd')):.1f} us")
print(f"copy 48MiB (torch): {timeit(lambda: x.clone()):.1f} us")

"""Bucket-order copy kernels at cfg2 (diagnostics): gather (read random rows, write
sequential) vs permute (read sequential, write random rows), GB/s of algorithmic bytes."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_01160_b200 import _lib  # noqa: E402
from paper_2306_01160_b200 import hash_sparse as hs  # noqa: E402

B, T, H, D, nb = 4, 8192, 12, 64, 16
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
q, k, v = (torch.randn((B, T, H, D), device=dev, generator=g).to(torch.bfloat16) for _ in range(3))
ids = torch.randint(0, nb, (B, T, H), device=dev, generator=g)
err = torch.zeros(1, dtype=torch.int32, device=dev)
hv, sb_, st_, sh_ = hs._hash_view(ids, B, H, T, "bth")
perm, rank, prob = hs._prepare_shared(hv, sb_, st_, sh_, B, H, T, D, err, True)


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


outs = [torch.empty((B, H, T, D), dtype=torch.bfloat16, device=dev) for _ in range(3)]
strides = []
for x in (q, k, v):
    strides += [x.stride(0), x.stride(1), x.stride(2)]


def gather():
    hs._gather3([q, k, v], [perm, perm, perm], "bthd")


def permute():
    _lib.call("scfa_permute_rows3", 3, _lib.ptr_array([q, k, v]), _lib.ptr_array(outs), _lib.ptr_array([rank] * 3),
              _lib.i64_array(strides), 2, B, T, H, D, _lib.i64_array([T] * 3), _lib.stream_ptr())


byts = 3 * 2 * B * T * H * D * 2
for name, fn in (("gather3", gather), ("permute3", permute)):
    ms = timed(fn)
    print(f"{name}: {ms * 1e3:.1f} us  {byts / ms / 1e6:.0f} GB/s")
ref = hs._gather3([q, k, v], [perm, perm, perm], "bthd")
permute()
torch.cuda.synchronize()
print("permute == gather:", all(torch.equal(a, b) for a, b in zip(ref, outs)))

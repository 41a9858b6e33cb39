"""cfg2 K/V permute: bucket ranks vs identity ranks vs a plain copy of the same bytes (diagnostics)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from permute_iso import timeit, k, v, rank, B, T, H, D, dev
from paper_2306_01160_b200 import hash_sparse as hs

ident = torch.arange(T, device=dev, dtype=torch.int32).repeat(B * H, 1).contiguous()
rnd = torch.argsort(torch.rand((B * H, T), device=dev), dim=1).to(torch.int32).contiguous()
nbytes = 2 * 2 * k.numel() * 2
for name, r in (("bucket", rank), ("identity", ident), ("random", rnd)):
    us = timeit(lambda: hs._permute3([k, v], [r, r], T))
    print(f"permute K,V {name}: {us:.1f} us  {nbytes / us / 1e3:.0f} GB/s")
ko, vo = torch.empty_like(k), torch.empty_like(v)
def cp():
    ko.copy_(k); vo.copy_(v)
us = timeit(cp)
print(f"copy_ K,V: {us:.1f} us  {nbytes / us / 1e3:.0f} GB/s")
kt = k.transpose(1, 2)
def tr():
    ko.view(B, H, T, D).copy_(kt); vo.view(B, H, T, D).copy_(v.transpose(1, 2))
us = timeit(tr)
print(f"transpose copy K,V: {us:.1f} us  {nbytes / us / 1e3:.0f} GB/s")

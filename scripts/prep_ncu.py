"""One cfg2 hash preparation (sort + finish + tile lists) for ncu (diagnostics)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_01160_b200 import hash_sparse as hs  # noqa: E402

B, T, H, D, nb = 4, 8192, 12, 64, 16
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
ids = torch.randint(0, nb, (B, T, H), device=dev, generator=g)
err = torch.zeros(1, dtype=torch.int32, device=dev)
for _ in range(2):
    hv, sb_, st_, sh_ = hs._hash_view(ids, B, H, T, "bth")
    perm, rank, prob = hs._prepare_shared(hv, sb_, st_, sh_, B, H, T, D, err, True)
    prob.schedule("fwd", "dq", "dkdv")
torch.cuda.synchronize()

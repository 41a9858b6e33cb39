import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2306_01160_b200 import hash_sparse as hs
B, T, H, D = 4, 8192, 12, 64
dev = torch.device("cuda")
h = torch.randint(0, 16, (B, T, H), device=dev)
err = torch.zeros(1, dtype=torch.int32, device=dev)
for _ in range(3):
    hs._prepare_shared(h, h.stride(0), h.stride(1), h.stride(2), B, H, T, D, err, True)
torch.cuda.synchronize()

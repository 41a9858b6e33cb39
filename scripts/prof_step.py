"""One cfg2 hash fwd+bwd step, repeated (a short command to run under ncu, needs a GPU).

    python scripts/prof_step.py [steps] [--single-pass] [--T 16384]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import bench
from paper_2306_01160_b200 import hash_sparse as hs

steps = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 3
sp = "--single-pass" in sys.argv
cfg = dict(bench.CFG)
if "--T" in sys.argv:
    cfg["T"] = int(sys.argv[sys.argv.index("--T") + 1])
qkvd, buckets = bench.make_inputs(cfg)
dev = torch.device("cuda")
q, k, v, dO = (torch.from_numpy(x).to(dev, torch.bfloat16) for x in qkvd)
hb = torch.from_numpy(buckets).to(dev)
for _ in range(steps):
    hs._fwd_bwd(q, k, v, hb, hb, dO, exclude_self=True, single_pass=sp)
torch.cuda.synchronize()
print("done", steps, "steps", "single-pass" if sp else "two-pass")

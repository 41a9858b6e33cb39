"""In-kernel per-tile clock64 stamps of the single-pass backward at cfg2 (diagnostics, GPU).

Row threads: 0 before the s_full wait, 1 after it, 10 after the ds_free wait, 2 after
p_full.  MMA lane: 6 loop top, 7 after the y / p_free waits, 3 after the S issue, 5 after
the previous tile's flush; in the flush: 12 start, 13 p_full seen, 4 dq_free seen.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import bench
from paper_2306_01160_b200 import _lib, hash_sparse as hs

TILES, SLOTS = 512, 16
cfg = dict(bench.CFG)
qkvd, buckets = bench.make_inputs(cfg)
dev = torch.device("cuda")
q, k, v, dO = (torch.from_numpy(x).to(dev, torch.bfloat16) for x in qkvd)
hb = torch.from_numpy(buckets).to(dev)
DET = "--det" in sys.argv  # two-pass dK/dV kernel instead of the single pass
KERNEL = "scfa_attn_bwd_dkdv" if DET else "scfa_attn_bwd"
for _ in range(3):
    hs._fwd_bwd(q, k, v, hb, hb, dO, single_pass=not DET)
torch.cuda.synchronize()
lib = _lib.load()
grid = 148
buf = torch.zeros(grid * TILES * SLOTS, dtype=torch.int64, device=dev)


def hook(name, phase):
    if name == KERNEL:
        lib.scfa_debug_timing(_lib.ptr(buf) if phase == 0 else None, TILES)


_lib.EVENT_HOOK = hook
hs._fwd_bwd(q, k, v, hb, hb, dO, single_pass=not DET)
torch.cuda.synchronize()
_lib.EVENT_HOOK = None
med = lambda x: float(np.median(x)) if len(x) else float("nan")
d = buf.view(grid, TILES, SLOTS).cpu().numpy().astype(np.float64)
for cta in (0, 1, 70, 147):
    r = d[cta]
    n = int((r[:, 6] > 0).sum())
    r = r[:n]
    per = np.diff(r[:, 6])
    print(f"cta {cta}: tiles {n}  span {r[-1, 5] - r[0, 6]:.0f} clk  period(mma loop) median {med(per):.0f}")
    print(f"   rows: s_wait {med(r[:, 1] - r[:, 0]):.0f}  ds_free wait {med(r[:, 10] - r[:, 1]):.0f}"
          f"  work {med(r[:, 2] - r[:, 10]):.0f}")
    print(f"   mma: wait_y/p_free {med(r[:, 7] - r[:, 6]):.0f}  issue_S {med(r[:, 3] - r[:, 7]):.0f}"
          f"  flush {med(r[:, 5] - r[:, 3]):.0f}  [flush: p_full wait {med(r[:, 13] - r[:, 12]):.0f}"
          f"  dq_free wait {med(r[:, 4] - r[:, 13]):.0f}]")
    print("   wait_y/p_free first 16:", (r[:16, 7] - r[:16, 6]).astype(int).tolist())
    print("   flush first 16:", (r[:16, 5] - r[:16, 3]).astype(int).tolist())
    print("   dq_free first 16:", (r[:16, 4] - r[:16, 13]).astype(int).tolist())
    print("   row s_wait first 16:", (r[:16, 1] - r[:16, 0]).astype(int).tolist())

"""In-kernel per-tile timestamps for the hash cfg2 forward/backward (diagnostics)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bench
from paper_2306_01160_b200 import _lib, hash_sparse as hs
from paper_2306_01160_b200._kernel import attention_forward, attention_backward

cfg = dict(bench.CFG)
qkvd, buckets = bench.make_inputs(cfg)
dev = torch.device("cuda")
q, k, v, dO = (torch.from_numpy(x).to(dev, torch.bfloat16) for x in qkvd)
hb = torch.from_numpy(buckets).to(dev)
T = cfg["T"]
sb = hs._sort_batch(q, k, v, hb, hb, "bthd", check=False)
prob = hs._problem_of(sb, True)
for _ in range(3):
    out = attention_forward(prob, sb.q, sb.k, sb.v, boundary=(T, False))
    g = attention_backward(prob, sb.q, sb.k, sb.v, out, dO, boundary=(T, T, False))
torch.cuda.synchronize()
TILES = 128
grid = 296
for name in ("fwd", "bwd"):
    buf = torch.zeros(grid * TILES * 8, dtype=torch.int64, device=dev)
    _lib.call("scfa_debug_timing", _lib.ptr(buf), TILES)
    if name == "fwd":
        out = attention_forward(prob, sb.q, sb.k, sb.v, boundary=(T, False))
    else:
        g = attention_backward(prob, sb.q, sb.k, sb.v, out, dO, boundary=(T, T, False))
    torch.cuda.synchronize()
    _lib.call("scfa_debug_timing", None, 0)
    d = buf.view(grid, TILES, 8).cpu().numpy().astype(np.float64)
    for cta in (0, 1, 150):
        rows = d[cta]
        n = int((rows[:, 0] > 0).sum())
        r = rows[:n]
        if n < 3:
            continue
        comp_wait = r[:, 1] - r[:, 0]
        softmax = r[:, 2] - r[:, 1]
        mma_wait_p = r[:, 4] - r[:, 3]
        mma_wait_y = r[:, 7] - r[:, 6]
        period = np.diff(r[:, 0])
        print(f"{name} cta {cta}: tiles {n}  period med {np.median(period):.0f}  comp_wait(s_full) med {np.median(comp_wait):.0f}"
              f"  softmax med {np.median(softmax):.0f}  mma_wait_p med {np.median(mma_wait_p):.0f}"
              f"  mma_wait_y med {np.median(mma_wait_y):.0f} max {mma_wait_y.max():.0f}")
        print("   first 12 periods:", period[:12].astype(int).tolist())
        print("   first 12 y waits:", mma_wait_y[:12].astype(int).tolist())
        print("   first 12 s waits:", comp_wait[:12].astype(int).tolist())

"""In-kernel per-tile clock64 stamps for the cfg2 hash step (diagnostics, needs a GPU).

Slots per tile (scfa_attn.cu SCFA_STAMP*): row thread 0: 0 before the s_full wait,
1 after it, 2 after p_full; 4 epilogue start (after acc_full, on the item's last
tile), 8 epilogue end.  MMA lane: 6 loop top, 7 after y/s_free waits, 3 after the S
issue, 5 after the previous tile's accumulate, 9 after x_full (item's first tile),
11 after the item's last accumulate.  Producer: 10 stationary-tile TMA issue.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import bench
from paper_2306_01160_b200 import _lib, hash_sparse as hs
from paper_2306_01160_b200._kernel import attention_backward, attention_forward

TILES = 160
SLOTS = 16

cfg = dict(bench.CFG)
qkvd, buckets = bench.make_inputs(cfg)
dev = torch.device("cuda")
q, k, v, dO = (torch.from_numpy(x).to(dev, torch.bfloat16) for x in qkvd)
hb = torch.from_numpy(buckets).to(dev)
T = cfg["T"]
sb = hs._sort_batch(q, k, v, hb, hb, "bthd", check=False)
prob = hs._problem_of(sb, True)
prob.schedule("fwd", "dq", "dkdv")
for _ in range(3):
    out = attention_forward(prob, sb.q, sb.k, sb.v, boundary=(T, False))
    g = attention_backward(prob, sb.q, sb.k, sb.v, out, dO, boundary=(T, T, False))
torch.cuda.synchronize()
lib = _lib.load()
grid = 148 * max(1, max(lib.scfa_debug_ctas_per_sm(m, 64) for m in range(3)))
bufs = {n: torch.zeros(grid * TILES * SLOTS, dtype=torch.int64, device=dev)
        for n in ("scfa_attn_fwd", "scfa_attn_bwd_dq", "scfa_attn_bwd_dkdv")}


def hook(name, phase):
    if name in bufs:
        lib.scfa_debug_timing(_lib.ptr(bufs[name]) if phase == 0 else None, TILES)


_lib.EVENT_HOOK = hook
out = attention_forward(prob, sb.q, sb.k, sb.v, boundary=(T, False))
g = attention_backward(prob, sb.q, sb.k, sb.v, out, dO, boundary=(T, T, False))
torch.cuda.synchronize()
_lib.EVENT_HOOK = None
print("ctas/sm", [lib.scfa_debug_ctas_per_sm(m, 64) for m in range(3)])

med = lambda x: float(np.median(x)) if len(x) else float("nan")
for name, buf in bufs.items():
    d = buf.view(grid, TILES, SLOTS).cpu().numpy().astype(np.float64)
    for cta in (0, 1, grid // 2):
        r = d[cta]
        n = int((r[:, 0] > 0).sum())
        r = r[:n]
        if n < 3:
            continue
        last = np.flatnonzero(r[:, 4] > 0)  # last tile of each item
        first = np.flatnonzero(r[:, 9] > 0)  # first tile of each item
        inner = np.setdiff1d(np.arange(n - 1), last)
        per = np.diff(r[:, 0])
        print(f"{name} cta {cta}: tiles {n} items {len(last)}  period(inner) {med(per[inner]):.0f}"
              f"  period(boundary) {med(per[last[last < n - 1]]):.0f}  s_wait {med(r[:, 1] - r[:, 0]):.0f}"
              f"  rows {med(r[:, 2] - r[:, 1]):.0f}")
        print(f"   boundary: acc_wait {med(r[last, 4] - r[last, 2]):.0f}  epilogue {med(r[last, 8] - r[last, 4]):.0f}"
              f"  next s_wait {med(r[last[last < n - 1] + 1, 1] - r[last[last < n - 1] + 1, 0]):.0f}"
              f"  gap->next tile {med(r[last[last < n - 1] + 1, 0] - r[last[last < n - 1], 8]):.0f}")
        print(f"   mma: wait_y/free {med(r[:, 7] - r[:, 6]):.0f}  issue_S {med(r[:, 3] - r[:, 7]):.0f}"
              f"  flush {med(r[:, 5] - r[:, 3]):.0f}  last-acc after p_full {med(r[last, 11] - r[last, 2]):.0f}"
              f"  x_full after X issue {med(r[first, 9] - r[first, 10]):.0f}")
        print("   periods:", per[:14].astype(int).tolist())
        # producer / flush detail (absolute clocks relative to the row threads' p_full stamp 2)
        rel = lambda a, b: med(r[:, a] - r[:, b])
        print(f"   K issue - s_full(row wait end) {rel(14, 1):.0f}  V issue - p_full {rel(15, 2):.0f}"
              f"  flush y1-ready - p_full {rel(12, 2):.0f}  flush p_full seen - p_full {rel(13, 2):.0f}")
        lr = lambda a, b: med(r[last, a] - r[last, b])
        print(f"   last tile: y1-ready - p_full {lr(12, 2):.0f}  p_full seen - p_full {lr(13, 2):.0f}"
              f"  issued(11) - seen(13) {lr(11, 13):.0f}  acc seen(4) - issued(11) {lr(4, 11):.0f}"
              f"  V issue(15) - p_full {lr(15, 2):.0f}")

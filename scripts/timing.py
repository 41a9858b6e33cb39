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

TILES = 512
SLOTS = 16

MODE = sys.argv[1] if len(sys.argv) > 1 else "hash"
cfg = dict(bench.CFG)
qkvd, buckets = bench.make_inputs(cfg)
dev = torch.device("cuda")
q, k, v, dO = (torch.from_numpy(x).to(dev, torch.bfloat16) for x in qkvd)
hb = torch.from_numpy(buckets).to(dev)
T = cfg["T"]
if MODE == "dense":
    from paper_2306_01160_b200.dense import causal_problem

    qe, ke, ve, de = (x.transpose(1, 2).contiguous() for x in (q, k, v, dO))
    prob = causal_problem(cfg["B"], cfg["H"], T, cfg["D"], dev)
    prob.schedule("fwd", "dq", "dkdv")

    class _SB:
        pass

    sb = _SB()
    sb.q, sb.k, sb.v = qe, ke, ve
    dO = de
    run = lambda: (attention_forward(prob, sb.q, sb.k, sb.v), None)
else:
    sb = hs._sort_batch(q, k, v, hb, hb, "bthd", check=False)
    prob = hs._problem_of(sb, True)
    prob.schedule("fwd", "dq", "dkdv")
bnd_f = None if MODE == "dense" else (T, False)
bnd_b = None if MODE == "dense" else (T, T, False)
for _ in range(3):
    out = attention_forward(prob, sb.q, sb.k, sb.v, boundary=bnd_f)
    g = attention_backward(prob, sb.q, sb.k, sb.v, out, dO, boundary=bnd_b)
torch.cuda.synchronize()
lib = _lib.load()
grid = 148 * max(1, max(lib.scfa_debug_ctas_per_sm(m, 64) for m in range(3)))
bufs = {n: torch.zeros(grid * TILES * SLOTS, dtype=torch.int64, device=dev)
        for n in ("scfa_attn_fwd", "scfa_attn_bwd_dq", "scfa_attn_bwd_dkdv")}


def hook(name, phase):
    if name in bufs:
        lib.scfa_debug_timing(_lib.ptr(bufs[name]) if phase == 0 else None, TILES)


_lib.EVENT_HOOK = hook
if MODE == "fused":  # the fused hash fwd+bwd (gathered stationary Q / dO, write-outs, fused delta)
    hs._fwd_bwd(q, k, v, hb, hb, dO)
else:
    out = attention_forward(prob, sb.q, sb.k, sb.v, boundary=bnd_f)
    g = attention_backward(prob, sb.q, sb.k, sb.v, out, dO, boundary=bnd_b)
torch.cuda.synchronize()
_lib.EVENT_HOOK = None
print("ctas/sm", [lib.scfa_debug_ctas_per_sm(m, 64) for m in range(3)])

os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"timing_{MODE}.npz"),
                    **{n: b.cpu().numpy() for n, b in bufs.items()},
                    ctas_per_sm=np.array([lib.scfa_debug_ctas_per_sm(m, 64) for m in range(3)]))
med = lambda x: float(np.median(x)) if len(x) else float("nan")
for name, buf in bufs.items():
    d = buf.view(grid, TILES, SLOTS).cpu().numpy().astype(np.float64)
    # whole-kernel view: per stream, first tile start .. last tile end (SM clocks differ per SM,
    # so only per-stream spans are comparable)
    spans, ntiles = [], []
    for c in range(grid):
        rr = d[c]
        m = rr[:, 0] > 0
        if m.sum() < 2:
            continue
        rr = rr[m]
        spans.append(rr[:, 2].max() - rr[:, 0].min())
        ntiles.append(len(rr))
    spans, ntiles = np.array(spans), np.array(ntiles)
    print(f"{name}: streams {len(spans)}  tiles/stream median {med(ntiles):.0f} max {ntiles.max()}"
          f"  span clk median {med(spans):.0f} max {spans.max():.0f}  (truncated at {TILES} tiles)")
    for cta in (0, 1, grid // 2):
        r = d[cta]
        n = int((r[:, 0] > 0).sum())
        r = r[:n]
        if n < 3:
            continue
        first = np.flatnonzero(r[:, 9] > 0)  # first tile of each item (MMA stamp)
        first = first[first > 0]
        last = first - 1
        inner = np.setdiff1d(np.arange(1, n), first)
        per = np.diff(r[:, 0])  # per[i] = stamp0(i+1) - stamp0(i)
        gap = r[1:n, 0] - r[:n - 1, 2]  # from a tile's p_full to the next tile's top
        print(f"{name} stream {cta}: tiles {n} items {len(first) + 1}  period(inner) {med(per[inner - 1]):.0f}"
              f"  period(item boundary) {med(per[first - 1]):.0f}  s_wait {med(r[:n, 1] - r[:n, 0]):.0f}"
              f"  rows {med(r[:n, 2] - r[:n, 1]):.0f}  gap(inner) {med(gap[inner - 1]):.0f}  gap(boundary) {med(gap[first - 1]):.0f}")
        print(f"   mma: wait_y/free {med(r[:n, 7] - r[:n, 6]):.0f}  issue_S {med(r[:n, 3] - r[:n, 7]):.0f}"
              f"  flush {med(r[:n, 5] - r[:n, 3]):.0f}")
        print("   periods:", per[:14].astype(int).tolist())
        L = last
        print(f"   boundary: p_full->handoff start {med(r[L, 4] - r[L, 2]):.0f}  barriers+ticket {med(r[L, 8] - r[L, 4]):.0f}"
              f"  queue wait {med(r[L, 10] - r[L, 8]):.0f}  write+arrive {med(r[L, 11] - r[L, 10]):.0f}"
              f"  handoff end->next tile {med(r[L + 1, 0] - r[L, 11]):.0f}")
        # producer / flush detail (absolute clocks relative to the row threads' p_full stamp 2)
        rel = lambda a, b: med(r[:, a] - r[:, b])
        print(f"   K issue - s_full(row wait end) {rel(14, 1):.0f}  V issue - p_full {rel(15, 2):.0f}"
              f"  flush y1-ready - p_full {rel(12, 2):.0f}  flush p_full seen - p_full {rel(13, 2):.0f}")


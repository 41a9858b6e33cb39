"""cfg2 step timeline: start / end of every entry point (CUDA events on the stream each is
launched on), relative to the step's first launch (diagnostics, needs a GPU).

The host queues the whole step behind a 2 ms device sleep, so the timeline is the GPU's,
not the launch loop's.  Prints the median over 10 steps.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import bench
from paper_2306_01160_b200 import _lib, hash_sparse as hs

cfg = dict(bench.CFG)
qkvd, buckets = bench.make_inputs(cfg)
dev = torch.device("cuda")
q, k, v, dO = (torch.from_numpy(x).to(dev, torch.bfloat16) for x in qkvd)
h = torch.from_numpy(buckets).to(dev)


def step():
    hs._fwd_bwd(q, k, v, h, h, dO, exclude_self=cfg["exclude_self"])


for _ in range(5):
    step()
torch.cuda.synchronize()
runs = []
for _ in range(10):
    log = []

    def hook(name, phase):
        e = torch.cuda.Event(enable_timing=True)
        e.record(torch.cuda.current_stream())
        log.append((name, phase, e))

    t0 = torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(4_000_000)
    t0.record()
    _lib.EVENT_HOOK = hook
    step()
    _lib.EVENT_HOOK = None
    t1 = torch.cuda.Event(enable_timing=True)
    t1.record()
    torch.cuda.synchronize()
    rows, open_ev = [], {}
    for name, phase, e in log:
        if phase == 0:
            open_ev[name] = e
        else:
            s = open_ev.pop(name)
            rows.append((name, t0.elapsed_time(s) * 1e3, t0.elapsed_time(e) * 1e3))
    rows.append(("(step end)", t0.elapsed_time(t1) * 1e3, t0.elapsed_time(t1) * 1e3))
    runs.append(rows)
names = [r[0] for r in runs[0]]
for i, n in enumerate(names):
    st = np.median([r[i][1] for r in runs])
    en = np.median([r[i][2] for r in runs])
    print(f"{n:28s} {st:8.1f} -> {en:8.1f} us  ({en - st:6.1f})")

"""Kernel-time breakdown of one cfg5 LM step per variant (torch.profiler / CUPTI).

  python scripts/profile_lm.py [--T 8192 --batch 4] [--variants hash,dense,sdpa]
"""

import argparse
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_01160_b200 import lm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=8192)
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--variants", default="hash,dense,sdpa")
    ap.add_argument("--rows", type=int, default=25)
    a = ap.parse_args()
    for v in a.variants.split(","):
        torch.manual_seed(0)
        model = lm.GPT(lm.LMConfig(attention=v, block_size=a.T)).cuda()
        opt = lm.make_optimizer(model)
        idx = torch.randint(0, 50304, (a.batch, a.T), device="cuda")
        tgt = torch.roll(idx, -1, 1)
        for _ in range(3):
            lm.train_step(model, opt, idx, tgt)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
            lm.train_step(model, opt, idx, tgt)
            torch.cuda.synchronize()
        print(f"===== {v} T={a.T} B={a.batch}")
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=a.rows, max_name_column_width=60))
        del model, opt
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

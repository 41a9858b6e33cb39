"""cfg5: GPT-2-small LM training step, H-LM (hash-sparse) vs F-LM (dense), 1 GPU.

  python scripts/bench_lm.py [--T 8192 --batch 4] [--steps 10 --warmup 3] [--variants hash,dense,sdpa]

Synthetic tokens, random init, bf16 autocast, AdamW step inside the timed region.
Per variant prints one JSON line: whole-step ms (CUDA events over the timed steps),
tokens/s, the last loss, parameter count and peak memory.
The paper's numbers (A100): H-LM iterations 1.8x (T=8192, nb=16) and
2.3x (T=16384) faster than F-LM.
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_01160_b200 import lm  # noqa: E402


def run(variant, T, batch, steps, warmup, nb):
    torch.manual_seed(0)
    cfg = lm.LMConfig(attention=variant, block_size=T, n_buckets=nb)
    model = lm.GPT(cfg).cuda()
    opt = lm.make_optimizer(model)
    g = torch.Generator(device="cuda").manual_seed(1)
    idx = torch.randint(0, cfg.vocab_size, (batch, T), device="cuda", generator=g)
    tgt = torch.roll(idx, -1, 1)
    for _ in range(warmup):
        lm.train_step(model, opt, idx, tgt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        loss = lm.train_step(model, opt, idx, tgt)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    out = {"variant": variant, "T": T, "batch": batch, "n_buckets": nb if variant == "hash" else None,
           "ms_per_step": round(ms, 3), "tokens_per_s": round(batch * T / ms * 1e3, 1), "loss": round(float(loss), 4),
           "params": model.n_params(), "peak_mem_gb": round(torch.cuda.max_memory_allocated() / 2**30, 2)}
    del model, opt
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=8192)
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--nb", type=int, default=16)
    ap.add_argument("--variants", default="hash,dense,sdpa")
    a = ap.parse_args()
    res = {}
    for v in a.variants.split(","):
        res[v] = run(v, a.T, a.batch, a.steps, a.warmup, a.nb)
        print(json.dumps(res[v]), flush=True)
    if "hash" in res and "dense" in res:
        print(json.dumps({"speedup_hash_vs_dense": round(res["dense"]["ms_per_step"] / res["hash"]["ms_per_step"], 3),
                          "speedup_hash_vs_sdpa": round(res["sdpa"]["ms_per_step"] / res["hash"]["ms_per_step"], 3)
                          if "sdpa" in res else None}))


if __name__ == "__main__":
    main()

"""BASELINE.json configs[2] and [3] on one B200: SCFA fwd+bwd sweeps next to dense causal attention.

  python scripts/sweep.py [--hash] [--qk] [--steps 10 --warmup 3] [--out gpurun_out/sweep.md]

hash (configs[3]): bucket count nb in 2..64 at T = 4k..32k, D = 64 / 128, H = 12,
  B * T = 32768 tokens per point (B = 8, 4, 2, 1).
qk (configs[2]): drop rate 0..90% of queries and keys per head at T = 16384, B = 4,
  H = 12, D = 64.

Per point: our fwd+bwd (the fused path bench.py times, inputs resident on the GPU,
CUDA events; hash and our dense comparator replay a CUDA graph as bench.py does — the
eager hash time is listed too —, and so does QK: its fused path sizes the compacted buffers
statically, with no host read-back), effective TFLOP/s on the visible (query, key) pairs (14 * D flops
per pair: fwd 4, dQ 6 incl. the recompute, dK/dV 4 ... as bench.py), our dense causal
comparator at the same shape, and torch's SDPA (cuDNN) dense causal fwd+bwd as a
library reference point.  Synthetic data: torch.randn Q/K/V/dO, uniform bucket ids /
Bernoulli keep masks.
"""

import argparse
import json
import os
import sys

import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2306_01160_b200 as scfa  # noqa: E402
from paper_2306_01160_b200 import hash_sparse as hs  # noqa: E402

dev = torch.device("cuda")


def timed(fn, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def timed_graph(fn, steps, warmup):
    """As timed(), replaying a CUDA graph of fn (paths with no host synchronisation)."""
    fn()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return timed(g.replay, steps, warmup)


def inputs(B, T, H, D, seed):
    g = torch.Generator(device=dev).manual_seed(seed)
    return [torch.randn((B, T, H, D), device=dev, generator=g).to(torch.bfloat16) for _ in range(4)]


_DENSE = {}


def dense_times(B, T, H, D, steps, warmup):
    key = (B, T, H, D)
    if key in _DENSE:
        return _DENSE[key]
    q, k, v, dO = inputs(B, T, H, D, 99)
    qe, ke, ve, de = (x.transpose(1, 2).contiguous() for x in (q, k, v, dO))

    def ours():
        o = scfa.flash_forward(qe, ke, ve, check=False)
        scfa.flash_backward(qe, ke, ve, o, de)

    qs, ks, vs = (x.clone().requires_grad_() for x in (qe, ke, ve))

    def sdpa():
        o = F.scaled_dot_product_attention(qs, ks, vs, is_causal=True)
        o.backward(de)

    r = (timed_graph(ours, steps, warmup), timed(sdpa, steps, warmup))
    del q, k, v, dO, qe, ke, ve, de, qs, ks, vs
    torch.cuda.empty_cache()
    _DENSE[key] = r
    return r


def hash_point(B, T, H, D, nb, steps, warmup):
    q, k, v, dO = inputs(B, T, H, D, nb)
    g = torch.Generator(device=dev).manual_seed(1000 + nb)
    ids = torch.randint(0, nb, (B, T, H), device=dev, generator=g)
    c = torch.nn.functional.one_hot(ids, nb).sum(1).to(torch.int64)  # (B, H, nb)
    p_live = int((c * (c - 1) // 2).sum())  # exclude_self
    f = lambda: hs._fwd_bwd(q, k, v, ids, ids, dO, exclude_self=True)
    eager = timed(f, steps, warmup)
    ms = timed_graph(f, steps, warmup)
    del q, k, v, dO
    torch.cuda.empty_cache()
    d_ours, d_sdpa = dense_times(B, T, H, D, steps, warmup)
    fl = 14.0 * D * p_live
    return {"kind": "hash", "B": B, "T": T, "H": H, "D": D, "nb": nb, "ms": round(ms, 4), "eager_ms": round(eager, 4),
            "eff_tflops": round(fl / ms / 1e9, 1), "dense_ms": round(d_ours, 4), "sdpa_ms": round(d_sdpa, 4),
            "speedup_vs_dense": round(d_ours / ms, 2), "speedup_vs_sdpa": round(d_sdpa / ms, 2)}


def qk_point(B, T, H, D, drop, steps, warmup):
    q, k, v, dO = inputs(B, T, H, D, int(drop * 100))
    qk = scfa.random_keep(B, T, H, drop, 6)
    kk = scfa.random_keep(B, T, H, drop, 7)
    qkd, kkd = torch.from_numpy(qk).to(dev), torch.from_numpy(kk).to(dev)
    kc = torch.cumsum(kkd > 0, dim=1)
    p_live = int(torch.where(qkd > 0, kc, torch.zeros_like(kc)).sum())
    # static compacted sizes (no host read-back): CUDA-graph replay, as bench.py's cfg3
    ms = timed_graph(lambda: scfa.qk_sparse_attention_fwd_bwd(q, k, v, qkd, kkd, dO, check=False), steps, warmup)
    del q, k, v, dO
    torch.cuda.empty_cache()
    d_ours, d_sdpa = dense_times(B, T, H, D, steps, warmup)
    fl = 14.0 * D * p_live
    return {"kind": "qk", "B": B, "T": T, "H": H, "D": D, "drop": drop, "ms": round(ms, 4),
            "eff_tflops": round(fl / ms / 1e9, 1), "dense_ms": round(d_ours, 4), "sdpa_ms": round(d_sdpa, 4),
            "speedup_vs_dense": round(d_ours / ms, 2), "speedup_vs_sdpa": round(d_sdpa / ms, 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hash", action="store_true")
    ap.add_argument("--qk", action="store_true")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default=None)
    ap.add_argument("--dims", type=lambda x: [int(d) for d in x.split(",")], default=[64, 128])
    a = ap.parse_args()
    if not (a.hash or a.qk):
        a.hash = a.qk = True
    rows = []
    if a.qk:
        for drop in (0.0, 0.1, 0.3, 0.5, 0.7, 0.9):
            rows.append(qk_point(4, 16384, 12, 64, drop, a.steps, a.warmup))
            print(json.dumps(rows[-1]), flush=True)
    if a.hash:
        for D in a.dims:
            for T, B in ((4096, 8), (8192, 4), (16384, 2), (32768, 1)):
                for nb in (2, 4, 8, 16, 32, 64):
                    rows.append(hash_point(B, T, 12, D, nb, a.steps, a.warmup))
                    print(json.dumps(rows[-1]), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            f.write("| kind | B | T | D | nb / drop | ours ms | eff TFLOP/s | dense (ours) ms | x dense | SDPA (cuDNN) ms "
                    "| x SDPA |\n|---|---|---|---|---|---|---|---|---|---|---|\n")
            for r in rows:
                p = r.get("nb", r.get("drop"))
                f.write(f"| {r['kind']} | {r['B']} | {r['T']} | {r['D']} | {p} | {r['ms']:.3f} | {r['eff_tflops']} | "
                        f"{r['dense_ms']:.3f} | {r['speedup_vs_dense']} | {r['sdpa_ms']:.3f} | {r['speedup_vs_sdpa']} |\n")


if __name__ == "__main__":
    main()

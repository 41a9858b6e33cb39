"""SCFA benchmark: hash-sparse fwd+bwd at cfg2 on B200, dense causal comparator, CPU baseline.

Contract (one JSON line on rank 0):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step = one pass of the hot path over one batch: bucket sort + fused
gather/transposes (prep), exact tile lists, forward, backward (dQ, dK/dV),
and the inverse scatters of O, dQ, dK, dV back to (B, T, H, D) (post).

Workload (BASELINE.json configs[1], "cfg2"): hash-sparse, B=4 H=12 T=8192
D=64, 16 buckets (same ids for Q and K, exclude_self on), bf16 operands,
fp32 gradients; synthetic inputs from the reference's seeded generators.
Metric: effective TFLOP/s = 14*D*P_live / t with P_live the number of
visible (query, key) pairs; ms per step is reported beside it.

Multi-GPU: one process per GPU.  `--gpus N` without a torchrun
environment re-launches itself under torch.distributed.run.  The 48 (b, h) units of
the cfg2 batch are partitioned across the ranks (sharding.shard_blocks: 48 / 24 / 12 / 6
units per rank at N = 1 / 2 / 4 / 8) with no collective on the data path: total work is
fixed ("scaling": "strong"); `value` = the whole batch's FLOPs / the max over ranks of
the per-rank CUDA-event step time.  NCCL is used for the max-over-ranks reduction and to
gather every rank's outputs and gradients to rank 0 for verification against rank 0's
own single-GPU run of the whole batch ("verify").  The replicated run (every rank its own
full cfg2 batch, weak scaling) is reported beside it when N > 1.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(workload="cfg2: hash-sparse SCFA fwd+bwd", B=4, H=12, T=8192, D=64, nb=16, exclude_self=True, seed=0)
METRIC = "SCFA fwd+bwd ms & effective TFLOP/s vs dense causal flash at T=8k/16k"
DATA = "synthetic (reference seeded generators: random_tensor seeds 0-3, random_buckets seed 5)"


def config_of(cfg, world):
    """The `config` dict of both arms (the same workload, whatever runs it)."""
    return {"workload": cfg["workload"], "B": cfg["B"], "H": cfg["H"], "T": cfg["T"], "D": cfg["D"],
            "buckets": cfg["nb"], "exclude_self": cfg["exclude_self"], "global_batch": cfg["B"],
            "parallelism": f"(b,h) units partitioned over {world} rank(s)" if world > 1 else "single device",
            "l2": "inputs > L2 (q,k,v,dO 4 x 48 MiB bf16 + sorted copies), no flush"}


def live_pairs_hash(buckets, exclude_self=True):
    """Visible pairs with shared Q/K bucket ids: sum_g c_g (c_g - 1) / 2 per head (+c_g without exclude_self)."""
    B, T, H = buckets.shape
    total = 0
    for b in range(B):
        for h in range(H):
            c = np.bincount(buckets[b, :, h]).astype(np.int64)
            total += int(np.sum(c * (c - 1) // 2 + (0 if exclude_self else c)))
    return total


def make_inputs(cfg):
    from paper_2306_01160_b200.hash_sparse import random_buckets
    from paper_2306_01160_b200.tensors import random_tensor_np

    B, H, T, D, s = cfg["B"], cfg["H"], cfg["T"], cfg["D"], cfg["seed"]
    shape = (B, H, T, D)
    # boundary layout (B, T, H, D), seeds s..s+3 and bucket seed s+5 as the reference CLI (cli.py:436-487)
    qkvd = [np.ascontiguousarray(np.swapaxes(random_tensor_np(shape, s + i, dtype=np.float32), 1, 2))
            for i in (0, 1, 2, 3)]
    buckets = random_buckets(B, T, H, cfg["nb"], s + 5)
    return qkvd, buckets


# ---------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) == 6:
                    self.rows.append(parts)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------- CPU baseline (oracle port)

def cpu_baseline(qkvd, buckets, cfg):
    """The reference tile loop restated in C (oracle/), all host threads, over every (b, h)
    head of the batch: the whole cfg2 step (sort + gather, fwd, bwd, scatter)."""
    from oracle import c_oracle

    c_oracle.build()
    threads = c_oracle.max_threads()
    B, H, T, D = cfg["B"], cfg["H"], cfg["T"], cfg["D"]
    q, k, v, d = qkvd
    heads = [(b, h) for b in range(B) for h in range(H)]
    excl = cfg["exclude_self"]

    t0 = time.perf_counter()
    hs = np.stack([buckets[b, :, h] for b, h in heads])  # (BH, T)
    order = np.argsort(hs * T + np.arange(T), axis=-1, kind="stable")  # reference _bucket_order
    take = lambda x: np.stack([x[b, :, h][order[i]] for i, (b, h) in enumerate(heads)])
    qs, ks, vs, ds = take(q), take(k), take(v), take(d)
    hsrt = np.take_along_axis(hs, order, -1)
    o, m, l, tiles = c_oracle.forward(qs, ks, vs, order, order, hsrt, hsrt, exclude_self=excl, threads=threads)
    dq, dk, dv = c_oracle.backward(qs, ks, vs, o, m, l, ds, order, order, hsrt, hsrt, exclude_self=excl,
                                   threads=threads)
    out = np.empty_like(o)
    np.put_along_axis(out, order[..., None], o, axis=1)  # hash_scatter
    elapsed = time.perf_counter() - t0

    flops = 14.0 * D * live_pairs_hash(buckets, excl)
    return {
        "value": flops / elapsed / 1e12,
        "unit": "TFLOP/s",
        "cores": threads,
        "kind": "port",
        "sample": f"the whole cfg2 step, all {B * H} (b,h) heads at T={T} D={D} nb={cfg['nb']}: sort+gather, fwd, "
                  f"bwd, scatter (oracle/scfa_oracle.c, fp32, 64x64 tiles), {elapsed:.2f} s",
        "seconds": elapsed,
        "ms_per_step": elapsed * 1e3,
    }


# ---------------------------------------------------------------- helpers

def live_pairs_qk(q_keep, k_keep):
    """Visible pairs of QK-sparse causal attention: per (b, h), sum over kept queries of the
    kept keys at or before them."""
    kc = np.cumsum(k_keep > 0, axis=1)  # kept keys at positions <= t
    return int(np.sum(np.where(q_keep > 0, kc, 0)))


class Ctx:
    """Per-rank plumbing: device, barrier, max over ranks, this rank's blocks."""

    def __init__(self, world, rank, local, dev):
        self.world, self.rank, self.local, self.dev = world, rank, local, dev

    def barrier(self):
        import torch
        import torch.distributed as dist

        if self.world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(self, x):
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=self.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def blocks(self, B, H):
        from paper_2306_01160_b200.sharding import shard_blocks

        return shard_blocks(B, H, self.rank, self.world)


def timed(ctx, fn, steps, warmup, graph=True):
    """CUDA-event time per step of fn (max over ranks), CUDA-graph replay unless graph=False."""
    import torch

    stream = torch.cuda.current_stream()
    run = fn
    if graph:
        fn()
        side = torch.cuda.Stream()
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            fn()
        stream.wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        run = g.replay
    for _ in range(warmup):
        run()
    ctx.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        run()
    e1.record(stream)
    ctx.barrier()
    return ctx.max_over_ranks(e0.elapsed_time(e1) / steps)


def measure_qk_cfg3(args, ctx, T=16384, drop=0.5):
    """BASELINE.json configs[2] at drop 0.5: QK-sparse fwd+bwd, B=4 H=12 T=16384 D=64, next to
    the dense causal comparator at the same shape; the (b, h) units partitioned like cfg2."""
    import torch

    import paper_2306_01160_b200 as scfa
    from paper_2306_01160_b200.sharding import slice_block

    B, H, D = 4, 12, 64
    gen = torch.Generator(device=ctx.dev).manual_seed(16)
    full = [torch.randn((B, T, H, D), device=ctx.dev, generator=gen).to(torch.bfloat16) for _ in range(4)]
    qk = scfa.random_keep(B, T, H, drop, 6)
    kk = scfa.random_keep(B, T, H, drop, 7)
    blocks = ctx.blocks(B, H)
    mine = [([slice_block(x, blk) for x in full],
             torch.from_numpy(np.ascontiguousarray(qk[blk[0]:blk[1], :, blk[2]:blk[3]])).to(ctx.dev),
             torch.from_numpy(np.ascontiguousarray(kk[blk[0]:blk[1], :, blk[2]:blk[3]])).to(ctx.dev)) for blk in blocks]
    del full
    p_live = live_pairs_qk(qk, kk)

    def step():
        for (q, k, v, dO), a, b in mine:
            scfa.qk_sparse_attention_fwd_bwd(q, k, v, a, b, dO, check=False)

    ms = timed(ctx, step, args.steps, args.warmup)
    eng = [[x.transpose(1, 2).contiguous() for x in xs] for xs, _, _ in mine]

    def dense():
        for qe, ke, ve, de in eng:
            o = scfa.flash_forward(qe, ke, ve, check=False)
            scfa.flash_backward(qe, ke, ve, o, de)

    dense_ms = timed(ctx, dense, args.steps, args.warmup)
    flops = 14.0 * D * p_live
    return {"workload": f"cfg3: QK-sparse SCFA fwd+bwd, B={B} H={H} T={T} D={D}, drop {drop}",
            "ms_per_step": ms, "effective_tflops": flops / (ms * 1e-3) / 1e12, "p_live": p_live,
            "dense_causal_ms": dense_ms,
            "dense_effective_tflops": 14.0 * D * B * H * T * (T + 1) / 2 / (dense_ms * 1e-3) / 1e12,
            "speedup_vs_dense": dense_ms / ms,
            "timing": "CUDA events over CUDA-graph replays, inputs resident (static compacted sizes: no host "
                      "read-back of the kept counts)"}


def measure_hash_t16k(args, ctx, B=4, H=12, T=16384, D=64, nb=16):
    """The north-star target shape for hash sparsity: fwd+bwd at T=16k with 16 buckets
    (B=4 H=12 D=64, as cfg3), next to the dense causal comparator at the same shape;
    CUDA-graph replay; (b, h) units partitioned like cfg2."""
    import torch

    import paper_2306_01160_b200 as scfa
    from paper_2306_01160_b200 import hash_sparse as hs
    from paper_2306_01160_b200.sharding import slice_block

    gen = torch.Generator(device=ctx.dev).manual_seed(17)
    full = [torch.randn((B, T, H, D), device=ctx.dev, generator=gen).to(torch.bfloat16) for _ in range(4)]
    ids = torch.randint(0, nb, (B, T, H), device=ctx.dev, generator=gen)
    c = torch.nn.functional.one_hot(ids, nb).sum(1).to(torch.int64)
    p_live = int((c * (c - 1) // 2).sum())
    mine = [([slice_block(x, blk) for x in full], slice_block(ids, blk)) for blk in ctx.blocks(B, H)]
    del full

    def step():
        for (q, k, v, dO), h in mine:
            hs._fwd_bwd(q, k, v, h, h, dO, exclude_self=True)

    ms = timed(ctx, step, args.steps, args.warmup)
    eng = [[x.transpose(1, 2).contiguous() for x in xs] for xs, _ in mine]

    def dense():
        for qe, ke, ve, de in eng:
            o = scfa.flash_forward(qe, ke, ve, check=False)
            scfa.flash_backward(qe, ke, ve, o, de)

    dense_ms = timed(ctx, dense, args.steps, args.warmup)
    return {"workload": f"hash-sparse SCFA fwd+bwd, B={B} H={H} T={T} D={D}, {nb} buckets (north-star target)",
            "ms_per_step": ms, "effective_tflops": 14.0 * D * p_live / (ms * 1e-3) / 1e12, "p_live": p_live,
            "dense_causal_ms": dense_ms, "speedup_vs_dense": dense_ms / ms,
            "timing": "CUDA events over CUDA-graph replays, inputs resident"}


# ---------------------------------------------------------------- host placement

def gpu_local_cpus(local):
    """Pin this process to the CPUs local to GPU `local` (the host buffers of the end-to-end
    leg are then first-touched on the GPU's NUMA node).  NVML first, then the PCI device's
    sysfs local_cpulist.  Returns a dict describing what happened (and the previous mask)."""
    import torch

    prev = os.sched_getaffinity(0)
    cpus, how = None, None
    try:
        import pynvml

        visible = (os.environ.get("CUDA_VISIBLE_DEVICES") or "").split(",")
        idx = int(visible[local]) if local < len(visible) and visible[local].strip().isdigit() else local
        pynvml.nvmlInit()
        try:
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        finally:
            pynvml.nvmlShutdown()
        cpus = {64 * w + b for w, m in enumerate(words) for b in range(64) if (int(m) >> b) & 1}
        how = "nvml"
    except Exception:
        cpus = None
    if not cpus:
        try:
            p = torch.cuda.get_device_properties(local)
            bdf = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            with open(f"/sys/bus/pci/devices/{bdf}/local_cpulist") as f:
                spec = f.read().strip()
            cpus = set()
            for part in spec.split(","):
                a, _, b = part.partition("-")
                cpus.update(range(int(a), int(b or a) + 1))
            how = f"sysfs {bdf}"
        except Exception:
            cpus = None
    info = {"prev": prev, "source": how, "local_cpus": len(cpus) if cpus else None, "allowed_cpus": len(prev)}
    if cpus:
        use = cpus & prev
        if use and use != prev:
            os.sched_setaffinity(0, use)
            info["pinned"] = len(use)
        else:
            info["pinned"] = "all allowed CPUs are GPU-local" if use else "no overlap with the allowed CPUs"
    else:
        info["pinned"] = "unknown locality"
    return info


def link_roofline(h2d_bytes, d2h_bytes, dev, reps=5):
    """Raw pinned copies of the e2e leg's byte counts: H2D alone, D2H alone and both at once
    on two streams (the e2e leg overlaps them); best of `reps`, CUDA events."""
    import torch

    src_h = torch.empty(h2d_bytes, dtype=torch.uint8, pin_memory=True)
    dst_d = torch.empty(h2d_bytes, dtype=torch.uint8, device=dev)
    src_d = torch.empty(d2h_bytes, dtype=torch.uint8, device=dev)
    dst_h = torch.empty(d2h_bytes, dtype=torch.uint8, pin_memory=True)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def t(fn):
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        return best

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            dst_d.copy_(src_h, non_blocking=True)
        with torch.cuda.stream(s2):
            dst_h.copy_(src_d, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    h2d_ms = t(lambda: dst_d.copy_(src_h, non_blocking=True))
    d2h_ms = t(lambda: dst_h.copy_(src_d, non_blocking=True))
    both_ms = t(both)
    return {"h2d_gbs": h2d_bytes / (h2d_ms * 1e-3) / 1e9, "d2h_gbs": d2h_bytes / (d2h_ms * 1e-3) / 1e9,
            "h2d_ms": h2d_ms, "d2h_ms": d2h_ms, "overlapped_ms": both_ms}


# ---------------------------------------------------------------- GPU arm

def prep_bytes(name, B, T, H, D, tiles_total, id_bytes=8):
    """Algorithmic HBM bytes of one preparation entry point, for its GB/s."""
    BH, T_pad = B * H, -(-T // 128) * 128
    if name == "scfa_hash_prepare":  # ids in; perm, rank, 5 slot vectors, 2 run vectors out
        return B * T * H * id_bytes + 2 * BH * T * 4 + 5 * BH * T_pad * 4 + 2 * BH * T_pad * 8
    if name == "scfa_permute_rows3":  # K, V rows: read in memory order, written to their slots
        return 2 * 2 * B * T * H * D * 2
    if name == "scfa_build_schedule":  # runs in; listed tiles (uint16) + counts out
        n_rb = -(-T // 128)
        return 2 * BH * T_pad * 8 + 2 * tiles_total + 3 * BH * n_rb * 4
    return None


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2306_01160_b200 as scfa
    from paper_2306_01160_b200 import _lib
    from paper_2306_01160_b200 import hash_sparse as hs
    from paper_2306_01160_b200.sharding import slice_block

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # diagnostics: SCFA_BENCH_SHARED_GPU=1 runs every rank on cuda:0 over gloo (the N > 1
    # plumbing exercised on a one-GPU box; the timing then means nothing)
    shared = world > 1 and os.environ.get("SCFA_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    _lib.require_cuda()
    ctx = Ctx(world, rank, local, dev)
    placement = gpu_local_cpus(local)

    qkvd, buckets = make_inputs(cfg)
    B, H, T, D = cfg["B"], cfg["H"], cfg["T"], cfg["D"]
    blocks = ctx.blocks(B, H)
    # this rank's units, boundary layout, pinned host copies (the e2e leg) and device copies
    host = [[slice_block(torch.from_numpy(x), blk).to(torch.bfloat16).pin_memory() for x in qkvd] for blk in blocks]
    host_h = [slice_block(torch.from_numpy(buckets), blk).pin_memory() for blk in blocks]
    dv_in = [[x.to(dev, non_blocking=True) for x in xs] for xs in host]
    dv_h = [h.to(dev, non_blocking=True) for h in host_h]
    torch.cuda.synchronize()
    p_live = live_pairs_hash(buckets, cfg["exclude_self"])
    flops_step = 14.0 * D * p_live  # the whole batch, all ranks
    my_units = sum((b1 - b0) * (h1 - h0) for b0, b1, h0, h1 in blocks)

    def step():
        res = []
        for (q, k, v, dO), h in zip(dv_in, dv_h):
            out, dq, dk, dv, prob = hs._fwd_bwd(q, k, v, h, h, dO, exclude_self=cfg["exclude_self"])
            res.append(((out.O, dq, dk, dv), prob))
        return res

    for _ in range(args.warmup):
        step()
    res = step()
    torch.cuda.synchronize()

    # verification: NCCL all_gather of every rank's outputs and gradients to rank 0,
    # compared with rank 0's own single-device run of the whole batch (bitwise: every
    # (b, h) slice is computed independently and the kernels are deterministic)
    verify = None
    if world > 1:
        verify = verify_gather(ctx, res, blocks, qkvd, buckets, cfg)

    # the step has no host synchronisation (hash mode: every size is static), so it is
    # captured once into a CUDA graph and replayed: the timed region holds K replays
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        step()
    torch.cuda.current_stream().wait_stream(side)
    launches0 = _lib.launches
    with torch.cuda.graph(graph):
        step()
    launches_per_step = _lib.launches - launches0
    for _ in range(args.warmup):
        graph.replay()
    stream = torch.cuda.current_stream()

    sampler = ClockSampler(local)
    with sampler:
        time.sleep(0.3)
        ctx.barrier()
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for _ in range(args.steps):
            graph.replay()
        t_end.record(stream)
        ctx.barrier()
    launches = launches_per_step * args.steps
    ms = ctx.max_over_ranks(t_start.elapsed_time(t_end) / args.steps)

    # per-entry-point CUDA events on the stream each entry point is launched on (the K / V
    # bucket-order copy runs on a side stream): the same K steps run eagerly
    ev_log = []

    def hook(name, phase):
        e = torch.cuda.Event(enable_timing=True)
        e.record(torch.cuda.current_stream())
        ev_log.append((name, phase, e))

    ctx.barrier()
    _lib.EVENT_HOOK = hook
    for _ in range(args.steps):
        step()
    _lib.EVENT_HOOK = None
    ctx.barrier()

    per = {}
    open_ev = {}
    for name, phase, e in ev_log:
        if phase == 0:
            open_ev[name] = e
        else:
            per.setdefault(name, []).append(open_ev.pop(name).elapsed_time(e))
    kern_ms = {n: sum(v) / args.steps for n, v in per.items()}
    kern_avg = {n: sum(v) / len(v) for n, v in per.items()}

    # end to end through the public API with host buffers: H2D inputs, D2H outputs + gradients
    outs_host = [[torch.empty(r.shape, dtype=r.dtype, pin_memory=True) for r in rr] for rr, _ in res]
    h2d = sum(x.numel() * x.element_size() for xs in host for x in xs) + sum(
        h.numel() * h.element_size() for h in host_h)
    d2h = sum(x.numel() * x.element_size() for xs in outs_host for x in xs)

    def e2e_step():
        # the public API on host tensors: per-batch-element streaming, H2D / compute / D2H
        # of consecutive elements overlapped; the results are on the host when it returns
        for xs, h, o in zip(host, host_h, outs_host):
            scfa.hash_sparse_attention_fwd_bwd(xs[0], xs[1], xs[2], h, h, xs[3], out=o)

    link_before = link_roofline(h2d, d2h, dev)
    for _ in range(args.warmup):
        e2e_step()
    e2e_each = []
    for _ in range(args.steps):  # each call returns with its results on the host
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        e2e_step()
        e1.record()
        torch.cuda.synchronize()
        e2e_each.append(e0.elapsed_time(e1))
    ctx.barrier()
    e2e_ms = ctx.max_over_ranks(sum(e2e_each) / len(e2e_each))
    link = link_roofline(h2d, d2h, dev)
    link["before_e2e_overlapped_ms"] = link_before["overlapped_ms"]

    # executed tiles per list, for tensor-pipe utilisation on executed tiles (this rank)
    tt = [0, 0, 0]
    for _, prob in res:
        for i, x in enumerate(prob._tiles_total.cpu().tolist()):
            tt[i] += x
    tiles = {"fwd_128x128": tt[0], "dq_128x64": tt[1], "dkdv_128x64": tt[2]}
    my_p_live = sum(live_pairs_hash(buckets[b0:b1, :, h0:h1], cfg["exclude_self"]) for b0, b1, h0, h1 in blocks)
    n_calls = len(blocks)
    algo = {"scfa_attn_fwd": 4.0 * D * my_p_live / n_calls, "scfa_attn_bwd_dq": 6.0 * D * my_p_live / n_calls,
            "scfa_attn_bwd_dkdv": 8.0 * D * my_p_live / n_calls}
    executed = {"scfa_attn_fwd": tt[0] * 128 * 128 * D * 2 * 2 / n_calls,
                "scfa_attn_bwd_dq": tt[1] * 128 * 64 * D * 2 * 3 / n_calls,
                "scfa_attn_bwd_dkdv": tt[2] * 128 * 64 * D * 2 * 4 / n_calls}
    attn = {n: kern_avg[n] for n in algo if n in kern_avg}
    dom = max(attn, key=lambda n: attn[n])
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    peak_src = "measured (MEASURED_PEAKS.json, burst)" if peaks else "fallback (B200_PROFILING.md)"
    peak = float(peaks.get("bf16_tflops", 1590.0))
    hbm = float(peaks.get("hbm_gbs", 6548.0))
    achieved = algo[dom] / (kern_avg[dom] * 1e-3) / 1e12
    traffic, traffic_src = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
        traffic, traffic_src = tj.get(dom), tj.get("_source")
    except OSError:
        pass
    roofline = {
        "bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak, "peak_source": peak_src,
        "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
        "traffic_source": traffic_src or "no committed ncu capture",
        "executed_tile_tflops": executed[dom] / (kern_avg[dom] * 1e-3) / 1e12,
        "executed_tile_frac": executed[dom] / (kern_avg[dom] * 1e-3) / 1e12 / peak,
        "per_kernel": {n: {"us": kern_avg[n] * 1e3, "achieved_tflops": algo[n] / (kern_avg[n] * 1e-3) / 1e12,
                           "frac": algo[n] / (kern_avg[n] * 1e-3) / 1e12 / peak,
                           "executed_tile_frac": executed[n] / (kern_avg[n] * 1e-3) / 1e12 / peak}
                       for n in attn},
    }
    # preparation kernels: algorithmic bytes / their own CUDA-event time, against HBM peak
    nbytes = {}
    for b0, b1, h0, h1 in blocks:
        for n in ("scfa_hash_prepare", "scfa_permute_rows3", "scfa_build_schedule"):
            x = prep_bytes(n, b1 - b0, T, h1 - h0, D, 0)
            nbytes[n] = nbytes.get(n, 0) + x
    nbytes["scfa_build_schedule"] += 2 * sum(tt)
    prep = {}
    for n, byt in nbytes.items():
        if n in kern_ms:
            gbs = byt / (kern_ms[n] * 1e-3) / 1e9
            prep[n] = {"us": kern_ms[n] * 1e3, "bytes": byt, "gbs": gbs, "frac_of_hbm": gbs / hbm}
    prep["_peak_gbs"] = hbm

    # the single-pass backward variant (scfa_attn_bwd: one key-stationary sweep, dQ reduced in
    # fp32) of the same step, for comparison with the default two-pass backward
    def step_single():
        for (q, k, v, dO), h in zip(dv_in, dv_h):
            hs._fwd_bwd(q, k, v, h, h, dO, exclude_self=cfg["exclude_self"], single_pass=True)

    sp_ms = timed(ctx, step_single, args.steps, args.warmup)

    # dense causal comparator at the same shape (our own kernels, engine layout, same fwd+bwd, same units)
    eng = [[x.transpose(1, 2).contiguous() for x in xs] for xs in dv_in]

    def dense():
        for qe, ke, ve, de in eng:
            o = scfa.flash_forward(qe, ke, ve, check=False)
            scfa.flash_backward(qe, ke, ve, o, de)

    dense_ms = timed(ctx, dense, args.steps, args.warmup)
    dense_flops = 14.0 * D * B * H * T * (T + 1) / 2
    cudnn = None
    if not args.no_cudnn:
        cudnn = measure_cudnn(args, ctx, eng)
    del eng

    cfg3 = None if args.no_cfg3 else measure_qk_cfg3(args, ctx)
    t16k = None if args.no_cfg3 else measure_hash_t16k(args, ctx)

    # weak scaling side field: every rank its own full cfg2 batch (replicated work)
    weak = None
    if world > 1 and not args.no_weak:
        full = [torch.from_numpy(x).to(dev, torch.bfloat16) for x in qkvd]
        hfull = torch.from_numpy(buckets).to(dev)
        wms = timed(ctx, lambda: hs._fwd_bwd(full[0], full[1], full[2], hfull, hfull, full[3],
                                             exclude_self=cfg["exclude_self"]), args.steps, args.warmup)
        weak = {"ms_per_step": wms, "value": world * flops_step / (wms * 1e-3) / 1e12, "unit": "TFLOP/s",
                "scaling": "weak", "global_batch": B * world,
                "note": "every rank runs its own full cfg2 batch (replicated inputs), max over ranks"}
        del full, hfull

    conf = config_of(cfg, world)
    conf.update({"units_per_rank": my_units, "blocks_rank0": blocks if rank == 0 else None,
                 "host_affinity": {k: v for k, v in placement.items() if k != "prev"}, "p_live": p_live})
    line = {
        "metric": METRIC,
        "value": flops_step / (ms * 1e-3) / 1e12,
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": DATA,
        "config": conf,
        "e2e": {"value": flops_step / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "paper_2306_01160_b200.hash_sparse_attention_fwd_bwd (host tensors, synchronous)",
                "link": link, "link_ms": link["overlapped_ms"],
                "frac_of_link": link["overlapped_ms"] / e2e_ms,
                "steps_ms": [round(x, 3) for x in e2e_each]},
        "gpu_launches": launches,
        "roofline": roofline,
        "prep": prep,
        "stages_ms": {n: round(v, 4) for n, v in sorted(kern_ms.items(), key=lambda kv: -kv[1])},
        "tiles": tiles,
        "single_pass_backward": {"ms_per_step": sp_ms, "value": flops_step / (sp_ms * 1e-3) / 1e12,
                                 "note": "same step with scfa_attn_bwd (dQ, dK, dV in one sweep; dQ by fp32 "
                                         "reductions, not bitwise reproducible); the headline uses the two-pass "
                                         "backward"},
        "dense_causal": {"ms_per_step": dense_ms, "effective_tflops": dense_flops / (dense_ms * 1e-3) / 1e12,
                         "speedup_of_scfa": dense_ms / ms},
        "clocks": sampler.summary(),
    }
    if cudnn is not None:
        line["cudnn_sdpa_causal"] = dict(cudnn, effective_tflops=dense_flops / (cudnn["ms_per_step"] * 1e-3) / 1e12,
                                         speedup_of_scfa=cudnn["ms_per_step"] / ms,
                                         our_dense_vs_cudnn=cudnn["ms_per_step"] / dense_ms)
    if verify is not None:
        line["verify"] = verify
    if weak is not None:
        line["weak"] = weak
    if cfg3 is not None:
        line["cfg3_qk"] = cfg3
    if t16k is not None:
        line["hash_t16k"] = t16k
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if placement.get("pinned") and isinstance(placement.get("pinned"), int):
            os.sched_setaffinity(0, placement["prev"])  # the CPU baseline gets every core again
        line["cpu_baseline"] = cpu_baseline(qkvd, buckets, cfg)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def measure_cudnn(args, ctx, eng):
    """torch SDPA (cuDNN / flash backend, a library comparator) causal fwd+bwd on the same
    engine-layout operands: is_causal=True, bf16, gradients in bf16."""
    import torch
    import torch.nn.functional as F

    ts = [[x.detach().clone().requires_grad_(i < 3) for i, x in enumerate(xs)] for xs in eng]

    def run():
        for q, k, v, d in ts:
            o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
            o.backward(d)
            q.grad = k.grad = v.grad = None

    try:
        with torch.nn.attention.sdpa_kernel([torch.nn.attention.SDPBackend.CUDNN_ATTENTION]):
            ms = timed(ctx, run, args.steps, args.warmup, graph=False)
        backend = "cudnn"
    except Exception:
        ms = timed(ctx, run, args.steps, args.warmup, graph=False)
        backend = "torch default"
    return {"ms_per_step": ms, "backend": backend}


def verify_gather(ctx, res, blocks, qkvd, buckets, cfg):
    """All-gather (NCCL, device tensors) every rank's O / dQ / dK / dV units to rank 0
    (sharding.gather_units) and compare them with rank 0's own run of the whole batch."""
    import torch
    import torch.distributed as dist

    from paper_2306_01160_b200 import hash_sparse as hs
    from paper_2306_01160_b200.sharding import gather_units

    B, H = cfg["B"], cfg["H"]
    full = gather_units([(blk, rr) for blk, (rr, _) in zip(blocks, res)], B, H)
    result = {"gathered": f"{dist.get_backend().upper()} all_gather of device tensors (O bf16, dQ/dK/dV fp32)",
              "world": ctx.world}
    if ctx.rank == 0:
        x = [torch.from_numpy(a).to(ctx.dev, torch.bfloat16) for a in qkvd]
        h = torch.from_numpy(buckets).to(ctx.dev)
        out, dq, dk, dv, _ = hs._fwd_bwd(x[0], x[1], x[2], h, h, x[3], exclude_self=cfg["exclude_self"])
        ok, worst = True, 0.0
        for got, want in zip(full, (out.O, dq, dk, dv)):
            ok &= bool(torch.equal(got, want))
            worst = max(worst, float((got.float() - want.float()).abs().max()))
        result.update({"bitwise_equal_to_single_device": ok, "max_abs_diff": worst})
    dist.barrier()
    return result


# ---------------------------------------------------------------- reference arm (CPU oracle port)

def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    qkvd, buckets = make_inputs(cfg)
    for _ in range(args.warmup):  # untimed steps (library load, page-in)
        cpu_baseline(qkvd, buckets, cfg)
    samples = [cpu_baseline(qkvd, buckets, cfg) for _ in range(max(1, args.steps))]
    vals = [s["value"] for s in samples]
    v = statistics.median(vals)
    base = dict(samples[0])
    base["value"] = v
    ms = statistics.median(s["ms_per_step"] for s in samples)
    line = {
        "metric": METRIC, "value": v, "unit": "TFLOP/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": DATA,
        "config": config_of(cfg, world),
        "cpu_baseline": base,
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "note": "the reference is NumPy (not installable as a native build here); its tile loop restated in C "
                "(oracle/scfa_oracle.c) runs the whole cfg2 step on the host cores, median of the timed steps",
    }
    print(json.dumps(line), flush=True)


def relaunch(args):
    """`--gpus N` outside torchrun: re-run this script under torch.distributed.run."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines show every rank
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.run(cmd, env=env).returncode)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cfg3", action="store_true", help="skip the T=16k side measurements")
    ap.add_argument("--no-cudnn", action="store_true", help="skip the torch SDPA (cuDNN) comparator")
    ap.add_argument("--no-weak", action="store_true", help="skip the replicated (weak scaling) side run")
    ap.add_argument("--T", type=int, default=None)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch(args)
    cfg = dict(CFG)
    if args.T:
        cfg["T"] = args.T
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()

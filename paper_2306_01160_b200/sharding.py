"""(b, h) sharding across ranks, one process per GPU.

Every (b, h) slice of the path is independent — index preparation is per (b, h)
along T (qk_sparse.py:59, hash_sparse.py:94) and the reference runs attention per
(b, h) through map_heads (tensors.py:178-189) — so the path shards with no
collective on the data path.  The B*H units are flattened and each rank takes one
contiguous range; a range is a list of segments (b, h0, h1), each a boundary-layout
slice x[b:b+1, :, h0:h1, :] that the rank runs as an independent call.  A
collective is used only to bring results to rank 0 for verification.
"""

import torch

__all__ = ["shard_segments", "shard_blocks", "slice_segment", "slice_block", "run_sharded", "gather_segments",
           "gather_units"]


def shard_segments(B, H, rank, world):
    """Contiguous range of the flattened (b, h) units owned by `rank`, as (b, h0, h1) segments."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    units = B * H
    u0, u1 = rank * units // world, (rank + 1) * units // world
    segs = []
    u = u0
    while u < u1:
        b, h0 = divmod(u, H)
        h1 = min(H, h0 + (u1 - u))
        segs.append((b, h0, h1))
        u += h1 - h0
    return segs


def shard_blocks(B, H, rank, world):
    """The same unit range as shard_segments, with runs of whole batch elements merged:
    a list of (b0, b1, h0, h1) blocks, each x[b0:b1, :, h0:h1] — whole heads of several
    batch elements (h0 = 0, h1 = H) or a head range of one.  Fewer, larger calls per rank
    (e.g. cfg2 over 2 ranks: one (B=2, H=12) block per rank instead of two segments)."""
    blocks = []
    for b, h0, h1 in shard_segments(B, H, rank, world):
        if blocks and h0 == 0 and h1 == H and blocks[-1][2] == 0 and blocks[-1][3] == H and blocks[-1][1] == b:
            blocks[-1] = (blocks[-1][0], b + 1, 0, H)
        else:
            blocks.append((b, b + 1, h0, h1))
    return blocks


def slice_block(x, blk):
    """Boundary-layout (B, T, H, ...) tensor -> its (b1-b0, T, h1-h0, ...) block (contiguous)."""
    b0, b1, h0, h1 = blk
    return x[b0:b1, :, h0:h1].contiguous()


def slice_segment(x, seg):
    """Boundary-layout (B, T, H, ...) tensor -> the segment's (1, T, h1-h0, ...) slice (contiguous)."""
    b, h0, h1 = seg
    return x[b:b + 1, :, h0:h1].contiguous()


def run_sharded(fn, tensors, rank, world):
    """Apply fn(*segment_slices) to each of this rank's segments.

    tensors: boundary-layout (B, T, H, ...) inputs; returns [(seg, fn result), ...].
    """
    B, _, H = tensors[0].shape[:3]
    return [(seg, fn(*[slice_segment(t, seg) for t in tensors])) for seg in shard_segments(B, H, rank, world)]


def gather_segments(results, shape, dtype, group=None, dst=0):
    """Assemble per-rank segment results into full (B, T, H, ...) tensors on rank `dst`.

    results: [(seg, (t0, t1, ...)), ...] from run_sharded with tuple-valued fn.  Uses
    torch.distributed all_gather_object (any backend: gloo on CPU, NCCL on GPUs);
    returns the list of full tensors on `dst`, None elsewhere.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group)
    payload = [(seg, [t.detach().cpu() for t in outs]) for seg, outs in results]
    everything = [None] * world
    dist.all_gather_object(everything, payload, group=group)
    if dist.get_rank(group) != dst:
        return None
    # a rank may own no segment (B*H < world): take the output count from any non-empty part
    n_out = next((len(part[0][1]) for part in everything if part), 0)
    full = [torch.zeros(shape, dtype=dtype) for _ in range(n_out)]
    for part in everything:
        for (b, h0, h1), outs in part:
            for f, o in zip(full, outs):
                f[b:b + 1, :, h0:h1] = o.to(dtype)
    return full


def gather_units(results, B, H, group=None, dst=0):
    """Collective gather of per-rank block results into full boundary-layout tensors on `dst`.

    results: [(block, (t0, t1, ...)), ...] for this rank's shard_blocks, each t_i a
    (b1-b0, T, h1-h0, ...) tensor.  Each output is packed as (units, T, ...) in unit order,
    padded to the largest rank's unit count and exchanged with dist.all_gather on the
    tensors' own device — NCCL over NVLink for CUDA tensors, gloo for CPU tensors — so no
    host round trip or pickling is involved.  Returns the full (B, T, H, ...) tensors on
    `dst`, None elsewhere.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    counts = [sum((b1 - b0) * (h1 - h0) for b0, b1, h0, h1 in shard_blocks(B, H, r, world)) for r in range(world)]
    mine = [r for _, r in results]
    n_out = len(mine[0]) if mine else None
    # every rank must agree on the number / dtypes / trailing shapes of the outputs
    meta = [None] * world
    dist.all_gather_object(meta, [(tuple(t.shape[1:2]) + tuple(t.shape[3:]), str(t.dtype)) for t in mine[0]]
                           if mine else None, group=group)
    ref = next(m for m in meta if m is not None)
    n_out = len(ref)
    umax = max(counts)
    full = []
    for i in range(n_out):
        tail, dt = ref[i]
        dtype = getattr(torch, dt.split(".")[-1])
        dev = mine[0][i].device if mine else (torch.device("cuda", torch.cuda.current_device())
                                               if dist.get_backend(group) == "nccl" else torch.device("cpu"))
        parts = [r[i].movedim(2, 1).reshape((-1,) + tail) for r in mine]  # (units, T, ...)
        buf = torch.zeros((umax,) + tail, dtype=dtype, device=dev)
        if parts:
            packed = torch.cat(parts)
            buf[: packed.shape[0]] = packed
        outs = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(outs, buf, group=group)
        if me == dst:
            allu = torch.cat([o[:c] for o, c in zip(outs, counts)])  # (B*H, T, ...)
            full.append(allu.reshape((B, H) + tail).movedim(1, 2).contiguous())
    return full if me == dst else None

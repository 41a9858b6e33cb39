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

__all__ = ["shard_segments", "slice_segment", "run_sharded", "gather_segments"]


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

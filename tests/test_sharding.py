"""(b, h) sharding across ranks: unit ranges, slices, and a world_size-2 gloo run on CPU.

The per-segment compute is the NumPy oracle (test infrastructure) so the multi-process
path — partition, independent per-segment calls, gather to rank 0 — is checked here
without a GPU; on GPUs the same helpers run with the CUDA path and NCCL.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import scfa_oracle as orc
from paper_2306_01160_b200.sharding import gather_segments, run_sharded, shard_segments


@pytest.mark.parametrize("B,H,world", [(4, 12, 1), (4, 12, 2), (4, 12, 8), (3, 5, 4), (2, 3, 7)])
def test_segments_partition_units(B, H, world):
    seen = []
    for r in range(world):
        for b, h0, h1 in shard_segments(B, H, r, world):
            assert 0 <= b < B and 0 <= h0 < h1 <= H
            seen += [b * H + h for h in range(h0, h1)]
    assert seen == list(range(B * H))  # contiguous, ordered, no overlap


def _hash_oracle(q, k, v, hsh):
    """(1, T, h, D) float64 slices -> oracle hash attention O (1, T, h, D), exclude_self."""
    T = q.shape[1]
    e = lambda x: np.swapaxes(x.numpy(), 1, 2)
    hh = hsh.numpy().transpose(0, 2, 1)
    pos = np.arange(T)
    vis = orc.visibility(pos, pos, hh, hh, exclude_self=True)
    O, _, _ = orc.attention(e(q), e(k), e(v), vis)
    return (torch.from_numpy(np.swapaxes(O, 1, 2)),)


def _worker(rank, world, port, q, k, v, hsh, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = run_sharded(_hash_oracle, [q, k, v, hsh], rank, world)
        full = gather_segments(res, q.shape, torch.float64)
        if rank == 0:
            out.copy_(full[0])
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_gloo_matches_single_process():
    B, T, H, D = 2, 96, 3, 16
    rng = np.random.default_rng(0)
    q, k, v = (torch.from_numpy(rng.standard_normal((B, T, H, D))) for _ in range(3))
    hsh = torch.from_numpy(rng.integers(0, 4, (B, T, H)))
    out = torch.zeros((B, T, H, D), dtype=torch.float64).share_memory_()
    mp.start_processes(_worker, args=(2, _free_port(), q, k, v, hsh, out), nprocs=2, join=True, start_method="fork")
    want = torch.cat([torch.cat([_hash_oracle(q[b:b + 1, :, h:h + 1], k[b:b + 1, :, h:h + 1], v[b:b + 1, :, h:h + 1],
                                              hsh[b:b + 1, :, h:h + 1])[0] for h in range(H)], dim=2)
                      for b in range(B)])
    assert torch.allclose(out, want, atol=1e-12)


def _worker_few(rank, world, port, q, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = run_sharded(lambda x: (2.0 * x,), [q], rank, world)
        full = gather_segments(res, q.shape, torch.float64)
        if rank == 0:
            out.copy_(full[0])
        else:
            assert full is None
    finally:
        dist.destroy_process_group()


def test_more_ranks_than_units_gathers():
    """B*H < world: some ranks own no segment, rank 0 among them possibly."""
    q = torch.arange(1 * 5 * 1 * 2, dtype=torch.float64).reshape(1, 5, 1, 2)
    out = torch.zeros_like(q).share_memory_()
    mp.start_processes(_worker_few, args=(3, _free_port(), q, out), nprocs=3, join=True, start_method="fork")
    assert torch.equal(out, 2.0 * q)


@pytest.mark.parametrize("B,H,world", [(4, 12, 1), (4, 12, 2), (4, 12, 3), (4, 12, 8), (3, 5, 4), (2, 3, 7)])
def test_blocks_cover_the_same_units(B, H, world):
    from paper_2306_01160_b200.sharding import shard_blocks

    for r in range(world):
        units = [b * H + h for b, h0, h1 in shard_segments(B, H, r, world) for h in range(h0, h1)]
        got = [b * H + h for b0, b1, h0, h1 in shard_blocks(B, H, r, world) for b in range(b0, b1) for h in range(h0, h1)]
        assert got == units
    if (B, H, world) == (4, 12, 2):
        assert shard_blocks(B, H, 0, world) == [(0, 2, 0, 12)]


def _worker_units(rank, world, port, x, out):
    from paper_2306_01160_b200.sharding import gather_units, shard_blocks, slice_block

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, T, H = x.shape[:3]
        res = [(blk, (slice_block(x, blk) * 3.0, slice_block(x, blk)[..., :1].to(torch.float32)))
               for blk in shard_blocks(B, H, rank, world)]
        full = gather_units(res, B, H)
        if rank == 0:
            out[0].copy_(full[0])
            out[1].copy_(full[1])
        else:
            assert full is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B,H,world", [(4, 12, 2), (2, 3, 4), (1, 2, 3)])
def test_gather_units_collective(B, H, world):
    """The bench's verification gather (all_gather of packed units) over gloo, uneven counts."""
    x = torch.randn((B, 7, H, 4), dtype=torch.float64)
    out = [torch.zeros_like(x).share_memory_(), torch.zeros((B, 7, H, 1), dtype=torch.float32).share_memory_()]
    mp.start_processes(_worker_units, args=(world, _free_port(), x, out), nprocs=world, join=True,
                       start_method="fork")
    assert torch.equal(out[0], 3.0 * x)
    assert torch.equal(out[1], x[..., :1].float())

"""The (b, h) partition on the CUDA path: every rank's blocks run as
independent calls, and the assembled results equal one call over the whole batch bit for
bit (the slices are independent, hash_sparse.py:94 / tensors.py:178-189, and the kernels
are deterministic).  The ranks are simulated in one process on cuda:0; the collective
that brings the blocks to rank 0 is tested over gloo in test_sharding.py and runs over
NCCL in bench.py --gpus N."""

import pytest
import torch

import paper_2306_01160_b200 as scfa
from paper_2306_01160_b200.sharding import shard_blocks, slice_block

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("kind", ["hash", "qk"])
def test_partitioned_blocks_equal_the_whole_batch(world, kind):
    B, T, H, D = 4, 1000, 6, 64
    g = torch.Generator(device="cuda").manual_seed(world)
    q, k, v, dO = (torch.randn((B, T, H, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    if kind == "hash":
        ids = torch.randint(0, 8, (B, T, H), device="cuda", generator=g)
        fn = lambda q_, k_, v_, a, d: scfa.hash_sparse_attention_fwd_bwd(q_, k_, v_, a, a, d)
        aux = ids
    else:
        keep = torch.from_numpy(scfa.random_keep(B, T, H, 0.5, world)).cuda()
        fn = lambda q_, k_, v_, a, d: scfa.qk_sparse_attention_fwd_bwd(q_, k_, v_, a, a, d)
        aux = keep
    want = fn(q, k, v, aux, dO)
    got = [torch.zeros_like(w) for w in want]
    for r in range(world):
        for blk in shard_blocks(B, H, r, world):
            b0, b1, h0, h1 = blk
            outs = fn(*(slice_block(x, blk) for x in (q, k, v, aux, dO)))
            for dst, o in zip(got, outs):
                dst[b0:b1, :, h0:h1] = o
    for name, a, b in zip(("O", "dQ", "dK", "dV"), got, want):
        assert torch.equal(a, b), name

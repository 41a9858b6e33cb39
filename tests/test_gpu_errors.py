"""The reference's error taxonomy on the fused and kernel-level calls (errors.py:4-29).

* NumericError when the output turns non-finite (update_stats, softmax.py:63-64): the
  forward kernel flags it in a device status word that every public call reads once
  after its launches are queued.
* ShapeError for negative bucket ids on the fused fwd+bwd (hash_sparse.py:112-113),
  which runs the sort without a host sync and reads the same status word.
* ShapeError for a dO whose shape differs from Q's (the reference backward's check).
* ContractError when a caller swaps the sorted vectors of a SortedBatch for unsorted ones
  (_check_sorted runs on every hash_forward_kernel call, hash_sparse.py:136-142).
"""

import dataclasses

import numpy as np
import pytest
import torch

import paper_2306_01160_b200 as scfa

pytestmark = pytest.mark.gpu


def _qkv(B=1, T=200, H=2, D=64, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return [torch.randn((B, T, H, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(4)]


def _ids(B=1, T=200, H=2, nb=4, seed=1):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randint(0, nb, (B, T, H), device="cuda", generator=g)


@pytest.mark.parametrize("bad", [float("nan"), float("inf")])
def test_hash_nonfinite_raises_numeric(bad):
    q, k, v, dO = _qkv()
    ids = _ids()
    v[0, 17, 1, 5] = bad
    with pytest.raises(scfa.NumericError):
        scfa.hash_sparse_attention(q, k, v, ids, ids)
    with pytest.raises(scfa.NumericError):
        scfa.hash_sparse_attention_fwd_bwd(q, k, v, ids, ids, dO)
    with pytest.raises(scfa.NumericError):
        scfa.dynamic_sparse_attention(q, k, v, ids, ids, sparsity_mode="hash")


def test_qk_and_dense_nonfinite_raise_numeric():
    q, k, v, dO = _qkv(T=256)
    q[0, 40, 0, 0] = float("nan")
    keep = scfa.random_keep(1, 256, 2, 0.3, 3)
    keep[0, 40, 0] = 1.0
    with pytest.raises(scfa.NumericError):
        scfa.qk_sparse_attention(q, k, v, keep, keep)
    with pytest.raises(scfa.NumericError):
        scfa.qk_sparse_attention_fwd_bwd(q, k, v, keep, keep, dO)
    qe, ke, ve = (x.transpose(1, 2).contiguous() for x in (q, k, v))
    with pytest.raises(scfa.NumericError):
        scfa.flash_forward(qe, ke, ve)


def test_nonfinite_in_invisible_rows_is_not_an_error():
    # a NaN key no query can see (dropped in QK mode) never reaches an output
    q, k, v, dO = _qkv(T=256)
    k[0, 50, 1, 3] = float("nan")
    keep = np.ones((1, 256, 2))
    keep[0, 50, 1] = 0.0
    o = scfa.qk_sparse_attention(q, k, v, keep, keep)
    assert bool(torch.isfinite(o.float()).all())


def test_fused_hash_rejects_negative_ids():
    q, k, v, dO = _qkv()
    ids = _ids()
    ids[0, 3, 1] = -2
    with pytest.raises(scfa.ShapeError):
        scfa.hash_sparse_attention_fwd_bwd(q, k, v, ids, ids, dO)
    with pytest.raises(scfa.ShapeError):
        scfa.hash_sparse_attention_autograd(q.requires_grad_(), k, v, ids, ids)


def test_fused_hash_rejects_large_ids():
    q, k, v, dO = _qkv()
    ids = _ids()
    ids[0, 9, 0] = 2 ** 31
    with pytest.raises(scfa.ShapeError):
        scfa.hash_sparse_attention_fwd_bwd(q, k, v, ids, ids, dO)


def test_fused_backward_checks_dout_shape():
    q, k, v, dO = _qkv()
    ids = _ids()
    short = dO[:, :150].contiguous()
    with pytest.raises(scfa.ShapeError):
        scfa.hash_sparse_attention_fwd_bwd(q, k, v, ids, ids, short)
    keep = scfa.random_keep(1, 200, 2, 0.5, 4)
    with pytest.raises(scfa.ShapeError):
        scfa.qk_sparse_attention_fwd_bwd(q, k, v, keep, keep, short)


def test_replaced_sorted_vectors_are_revalidated():
    qe, ke, ve = (torch.randn((1, 2, 200, 64), device="cuda").to(torch.bfloat16) for _ in range(3))
    h = torch.randint(0, 4, (1, 2, 200), device="cuda")
    sb = scfa.sort_by_bucket(qe, ke, ve, h, h)
    scfa.hash_forward_kernel(sb)  # the batch's own sorted vectors: fine
    bad = dataclasses.replace(sb, q_hash=sb.q_hash.flip(-1).contiguous())
    with pytest.raises(scfa.ContractError):
        scfa.hash_forward_kernel(bad)


def test_host_results_are_complete_on_return():
    # padded head dim + host inputs: the wrapper slices the host results right away
    B, T, H, D = 2, 1500, 3, 48
    g = torch.Generator().manual_seed(0)
    q, k, v, dO = (torch.randn((B, T, H, D), generator=g).to(torch.bfloat16) for _ in range(4))
    ids = torch.randint(0, 8, (B, T, H), generator=g)
    got = scfa.hash_sparse_attention_fwd_bwd(q, k, v, ids, ids, dO)
    want = scfa.hash_sparse_attention_fwd_bwd(*(x.cuda() for x in (q, k, v)), ids.cuda(), ids.cuda(), dO.cuda())
    for a, b in zip(got, want):
        assert not a.is_cuda
        assert torch.equal(a, b.cpu())


def test_contract_narrowing_at_the_boundary():
    """The engine's documented limits raise the reference's ShapeError: head dim > 128
    (the tcgen05 tiles take 64 / 128; the reference takes any D) and bucket ids >= 2**31
    (int32 keys; the reference sorts int64, hash_sparse.py:93-94)."""
    q, k, v, dO = _qkv(D=64)
    wide = torch.zeros((1, 200, 2, 160), device="cuda", dtype=torch.bfloat16)
    ids = _ids()
    with pytest.raises(scfa.ShapeError):
        scfa.hash_sparse_attention(wide, wide, wide, ids, ids)
    with pytest.raises(scfa.ShapeError):
        scfa.qk_sparse_attention(wide, wide, wide, torch.ones((1, 200, 2)), torch.ones((1, 200, 2)))
    big = ids.clone()
    big[0, 5, 0] = 2 ** 31
    qe, ke, ve = (x.transpose(1, 2).contiguous() for x in (q, k, v))
    with pytest.raises(scfa.ShapeError):
        scfa.sort_by_bucket(qe, ke, ve, big.transpose(1, 2), big.transpose(1, 2))
    with pytest.raises(scfa.ShapeError):
        scfa.hash_sparse_attention(q, k, v, big, big)

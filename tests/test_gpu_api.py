"""The reference's own kernel-level and end-to-end tests (pkg/tests/test_qk.py,
test_hash.py), restated on the CUDA path, mostly at D = 64 (the engine's tile head dims
are 64 / 128; other D <= 128 are zero-padded by the public calls — tested at the end,
including the reference's own D = 4).

Exact-equality tests (`bitwise dense`, `zero upstream`, `all dropped`, `collision
pattern`) keep the reference's exactness; numeric comparisons use the bf16 tolerance
of test_gpu_attention.py.
"""

import numpy as np
import pytest
import torch

import paper_2306_01160_b200 as scfa
from oracle import scfa_oracle as orc

from conftest import bf16_round, make_batch

pytestmark = pytest.mark.gpu


def _t(x, dtype=torch.bfloat16):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


def _np(x):
    return x.detach().float().cpu().numpy().astype(np.float64)


def _boundary(x):  # (B, H, T, D) -> (B, T, H, D)
    return np.ascontiguousarray(np.swapaxes(x, 1, 2))


# ------------------------------------------------------------------ QK (test_qk.py)

def test_qk_no_drops_is_bitwise_dense():  # test_qk.py:137-146
    q, k, v = (_t(x) for x in make_batch(2, 2, 300, 64, seed=5))
    dense = scfa.flash_forward(q, k, v)
    idx = torch.arange(300).expand(2, 2, 300)
    sparse = scfa.qk_forward_kernel(q, k, v, idx, idx)
    assert torch.equal(sparse.O, dense.O)
    assert torch.equal(sparse.M, dense.M) and torch.equal(sparse.L, dense.L)
    assert sparse.tiles_computed == dense.tiles_computed


def test_qk_no_drops_backward_matches_dense():  # test_qk.py:194-204
    q, k, v = (_t(x) for x in make_batch(1, 2, 200, 64, seed=15))
    d_out = _t(bf16_round(np.random.default_rng(17).standard_normal((1, 2, 200, 64))))
    dense_out = scfa.flash_forward(q, k, v)
    want = scfa.flash_backward(q, k, v, dense_out, d_out)
    idx = torch.arange(200).expand(1, 2, 200)
    out = scfa.qk_forward_kernel(q, k, v, idx, idx)
    got = scfa.qk_backward_kernel(q, k, v, out, d_out, idx, idx)
    for g, w in zip(got, want):
        assert torch.equal(g, w)


def test_qk_compacted_instance_visible_key_counts():  # test_qk.py:148-162
    # uniform logits + one-hot values: row i averages its visible keys
    q_idx = torch.tensor([0, 1, 2, 3, 6, 7]).view(1, 1, 6)
    k_idx = torch.tensor([0, 2, 3, 5, 6, 7]).view(1, 1, 6)
    q = torch.ones(1, 1, 6, 64)
    k = torch.ones(1, 1, 6, 64)
    v = torch.zeros(1, 1, 6, 64)
    v[0, 0, :, :6] = torch.eye(6)
    out = scfa.qk_forward_kernel(_t(q.numpy()), _t(k.numpy()), _t(v.numpy()), q_idx, k_idx)
    o = _np(out.O)[0, 0, :, :6]
    counts = (o > 0).sum(axis=1)
    assert counts.tolist() == [1, 1, 2, 3, 5, 6]
    nonzero = o[o > 0]
    assert np.allclose(nonzero, np.repeat(1.0 / counts, counts), rtol=1e-2)


def test_qk_contract_errors():  # test_qk.py:176-191
    q, k, v = (_t(x) for x in make_batch(1, 1, 4, 64, seed=13))
    good = torch.arange(4).view(1, 1, 4)
    bad = torch.tensor([2, 0, 1, 3]).view(1, 1, 4)
    interior = torch.tensor([0, scfa.QUERY_PAD, 2, 3]).view(1, 1, 4)
    for qi, ki in ((bad, good), (good, bad), (interior, good)):
        with pytest.raises(scfa.ContractError):
            scfa.qk_forward_kernel(q, k, v, qi, ki)


def test_qk_zero_upstream_gives_zero_gradients():  # test_qk.py:206-215
    qb, kb, vb = (_boundary(x) for x in make_batch(1, 1, 160, 64, seed=19))
    keep = scfa.random_keep(1, 160, 1, 0.3, 20)
    prep = scfa.qk_preprocess(_t(qb), _t(kb), _t(vb), keep, keep)
    out = scfa.qk_forward_kernel(prep.q_c, prep.k_c, prep.v_c, prep.q_idx, prep.k_idx)
    grads = scfa.qk_backward_kernel(prep.q_c, prep.k_c, prep.v_c, out, torch.zeros_like(prep.q_c), prep.q_idx,
                                    prep.k_idx)
    assert not any(bool(g.any()) for g in grads)


def test_qk_all_queries_or_keys_dropped():  # test_qk.py:261-276
    qb, kb, vb = (_boundary(x) for x in make_batch(1, 2, 160, 64, seed=29))
    none = np.zeros((1, 160, 2))
    some = scfa.random_keep(1, 160, 2, 0.3, 30)
    for qk_, kk_ in ((none, some), (some, none)):
        out = scfa.qk_sparse_attention(_t(qb), _t(kb), _t(vb), qk_, kk_)
        assert tuple(out.shape) == (1, 160, 2, 64)
        assert not bool(out.any()) and bool(torch.isfinite(out).all())
        o, gq, gk, gv = scfa.qk_sparse_attention_fwd_bwd(_t(qb), _t(kb), _t(vb), qk_, kk_, _t(qb))
        assert not any(bool(x.any()) for x in (o, gq, gk, gv))


def test_qk_all_keep_equals_dense():  # test_qk.py:254-259
    q, k, v = make_batch(2, 2, 300, 64, seed=27)
    keep = np.ones((2, 300, 2))
    got = scfa.qk_sparse_attention(_t(_boundary(q)), _t(_boundary(k)), _t(_boundary(v)), keep, keep)
    want = scfa.flash_forward(_t(q), _t(k), _t(v)).O
    assert torch.equal(got, want.transpose(1, 2))


# ------------------------------------------------------------------ hash (test_hash.py)

def test_lsh_antipodal_offset_and_determinism():  # test_hash.py:61-71
    x = torch.randn(2, 100, 3, 64, dtype=torch.float64)
    a = scfa.lsh_buckets(x, 16, 5)
    assert torch.equal(scfa.lsh_buckets(-x, 16, 5), (a + 8) % 16)
    assert torch.equal(scfa.lsh_buckets(x, 16, 5), a)
    assert not torch.equal(scfa.lsh_buckets(x, 16, 6), a)


def test_normalize_keys():  # test_hash.py:99-116
    q = torch.randn(1, 10, 2, 64, device="cuda")
    n = scfa.normalize_keys(q)
    assert torch.allclose(n.norm(dim=-1), torch.ones(1, 10, 2, device="cuda"), atol=1e-5)
    assert torch.allclose(scfa.normalize_keys(n), n, atol=1e-6)
    q[0, 3, 1] = 0
    with pytest.raises(scfa.NumericError):
        scfa.normalize_keys(q)


def test_hash_single_bucket_is_bitwise_dense():  # test_hash.py:209-219
    q, k, v = (_t(x) for x in make_batch(2, 2, 300, 64, seed=61))
    hashes = torch.zeros((2, 2, 300), dtype=torch.int64)
    sb = scfa.sort_by_bucket(q, k, v, hashes, hashes)
    out = scfa.hash_forward_kernel(sb, exclude_self=False)
    want = scfa.flash_forward(q, k, v)
    assert torch.equal(out.O, want.O)
    assert torch.equal(out.M, want.M) and torch.equal(out.L, want.L)
    assert out.tiles_computed == want.tiles_computed


def test_hash_earliest_in_bucket_is_zero_with_exclude_self():  # test_hash.py:221-230
    q, k, v = (_t(x) for x in make_batch(1, 1, 6, 64, seed=67))
    buckets = torch.tensor([0, 0, 0, 1, 1, 1]).view(1, 1, 6)
    sb = scfa.sort_by_bucket(q, k, v, buckets, buckets)
    out = scfa.hash_forward_kernel(sb, exclude_self=True)
    o = scfa.hash_scatter(out.O, sb.q_idx)
    assert not bool(o[0, 0, 0].any()) and not bool(o[0, 0, 3].any())
    assert bool(o[0, 0, 1].any()) and bool(torch.isfinite(o).all())


def test_hash_contract_error_on_unsorted_batch():  # test_hash.py:243-253
    q, k, v = (_t(x) for x in make_batch(1, 1, 6, 64, seed=79))
    buckets = torch.tensor([1, 0, 0, 1, 0, 1]).view(1, 1, 6)
    sb = scfa.sort_by_bucket(q, k, v, buckets, buckets)
    broken = scfa.SortedBatch(q=sb.q, k=sb.k, v=sb.v, q_idx=sb.q_idx, k_idx=sb.k_idx, q_hash=buckets.cuda(),
                              k_hash=sb.k_hash)
    with pytest.raises(scfa.ContractError):
        scfa.hash_forward_kernel(broken)


def test_hash_distinct_buckets_exclude_self_all_zero():  # test_hash.py:304-313
    T = 300
    qb, kb, vb = (_boundary(x) for x in make_batch(1, 2, T, 64, seed=127))
    buckets = np.broadcast_to(np.arange(T)[None, :, None], (1, T, 2)).copy()
    out = scfa.hash_sparse_attention(_t(qb), _t(kb), _t(vb), buckets, buckets, exclude_self=True)
    assert not bool(out.any()) and bool(torch.isfinite(out).all())


def test_hash_weight_pattern_is_exactly_collision_set():  # test_hash.py:328+
    # one-hot values expose the attention matrix: positive weights == same bucket and causal
    T, nb = 64, 4
    rng = np.random.default_rng(3)
    q = bf16_round(rng.standard_normal((1, T, 1, 64)) * 0.1)
    k = bf16_round(rng.standard_normal((1, T, 1, 64)) * 0.1)
    v = np.zeros((1, T, 1, 64))
    v[0, :, 0, :T] = np.eye(T)
    buckets = rng.integers(0, nb, (1, T, 1))
    out = _np(scfa.hash_sparse_attention(_t(q), _t(k), _t(v), buckets, buckets, exclude_self=False))
    w = out[0, :, 0, :T]
    b = buckets[0, :, 0]
    want = (b[:, None] == b[None, :]) & (np.arange(T)[None, :] <= np.arange(T)[:, None])
    assert np.array_equal(w > 0, want)


# ------------------------------------------------------------------ acceptance (test_acceptance.py)

def test_determinism():  # test_acceptance.py:415+ (atomic-free backward: bitwise repeatable)
    qb, kb, vb = (_boundary(x) for x in make_batch(2, 3, 777, 64, seed=41))
    dO = _t(bf16_round(np.random.default_rng(42).standard_normal((2, 777, 3, 64))))
    hb = _t(scfa.random_buckets(2, 777, 3, 8, 43), torch.int64)
    a = scfa.hash_sparse_attention_fwd_bwd(_t(qb), _t(kb), _t(vb), hb, hb, dO)
    b = scfa.hash_sparse_attention_fwd_bwd(_t(qb), _t(kb), _t(vb), hb, hb, dO)
    for x, y in zip(a, b):
        assert torch.equal(x, y)


def test_nan_safety_large_logits():  # test_acceptance.py:203+
    qb, kb, vb = (_boundary(x) for x in make_batch(1, 2, 256, 64, seed=47))
    qb = qb * 60.0  # logits far beyond exp range before max subtraction
    keep = scfa.random_keep(1, 256, 2, 0.5, 48)
    o, gq, gk, gv = scfa.qk_sparse_attention_fwd_bwd(_t(qb), _t(kb), _t(vb), keep, keep, _t(qb))
    assert all(bool(torch.isfinite(x).all()) for x in (o, gq, gk, gv))
    hb = scfa.random_buckets(1, 256, 2, 4, 49)
    o, gq, gk, gv = scfa.hash_sparse_attention_fwd_bwd(_t(qb), _t(kb), _t(vb), hb, hb, _t(qb))
    assert all(bool(torch.isfinite(x).all()) for x in (o, gq, gk, gv))


# ------------------------------------------------------------------ head dims other than 64 / 128

@pytest.mark.parametrize("D", [4, 8, 32, 96])
def test_small_and_odd_head_dims_match_oracle(D):
    """The engine zero-pads D up to 64 / 128 (scale stays 1/sqrt(D)): same results as the
    oracle at the caller's D, for the end-to-end hash and QK fwd+bwd and the dense path."""
    B, H, T = 1, 2, 200
    qb, kb, vb = (_boundary(x) for x in make_batch(B, H, T, D, seed=91))
    dO = bf16_round(np.random.default_rng(92).standard_normal((B, T, H, D)))
    eng = lambda x: np.swapaxes(x, 1, 2)
    hb = scfa.random_buckets(B, T, H, 4, 93)
    hh = hb.transpose(0, 2, 1)
    pos = np.arange(T)
    vis = orc.visibility(pos, pos, hh, hh, exclude_self=True)
    O, _, _ = orc.attention(eng(qb), eng(kb), eng(vb), vis)
    grads = orc.attention_grads(eng(qb), eng(kb), eng(vb), vis, eng(dO))
    got = scfa.hash_sparse_attention_fwd_bwd(_t(qb), _t(kb), _t(vb), _t(hb, torch.int64), _t(hb, torch.int64),
                                             _t(dO))
    for g, w in zip(got, (O,) + tuple(grads)):
        assert g.shape[-1] == D
        assert np.max(np.abs(_np(g) - eng(w))) <= 2e-2
    o = scfa.hash_sparse_attention(_t(qb), _t(kb), _t(vb), hb, hb)
    assert tuple(o.shape) == (B, T, H, D) and np.max(np.abs(_np(o) - eng(O))) <= 2e-2
    # dense comparator, kernel level
    q, k, v = (_t(eng(x)) for x in (qb, kb, vb))
    out = scfa.flash_forward(q, k, v)
    Od, _, _ = orc.attention(eng(qb), eng(kb), eng(vb), orc.visibility(pos, pos))
    assert out.O.shape[-1] == D and np.max(np.abs(_np(out.O) - Od)) <= 2e-2
    gd = scfa.flash_backward(q, k, v, out, _t(eng(dO)))
    wd = orc.attention_grads(eng(qb), eng(kb), eng(vb), orc.visibility(pos, pos), eng(dO))
    for g, w in zip(gd, wd):
        assert g.shape[-1] == D and np.max(np.abs(_np(g) - w)) <= 2e-2


def test_reference_style_tiny_head_dim_bitwise_dense():  # test_qk.py:137-146 at its own D = 4
    q, k, v = (_t(x) for x in make_batch(2, 2, 48, 4, seed=5))
    dense = scfa.flash_forward(q, k, v)
    idx = torch.arange(48).expand(2, 2, 48)
    sparse = scfa.qk_forward_kernel(q, k, v, idx, idx)
    assert sparse.O.shape[-1] == 4
    assert torch.equal(sparse.O, dense.O) and torch.equal(sparse.M, dense.M)


def test_autograd_with_padded_head_dim():
    B, T, H, D = 1, 256, 2, 40
    rng = np.random.default_rng(94)
    x = [torch.from_numpy(rng.standard_normal((B, T, H, D)).astype(np.float32)).cuda().requires_grad_()
         for _ in range(3)]
    ids = torch.from_numpy(scfa.random_buckets(B, T, H, 4, 95)).cuda()
    o = scfa.dynamic_sparse_attention(x[0], x[1], x[2], ids, ids)
    assert o.shape[-1] == D
    o.sum().backward()
    assert all(t.grad is not None and t.grad.shape[-1] == D and bool(torch.isfinite(t.grad).all()) for t in x)
    with pytest.raises(scfa.ShapeError):
        scfa.hash_sparse_attention(torch.zeros(1, 8, 1, 160), torch.zeros(1, 8, 1, 160), torch.zeros(1, 8, 1, 160),
                                   ids[:, :8, :1], ids[:, :8, :1])

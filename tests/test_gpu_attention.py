"""GPU parity: the tcgen05 kernels against the NumPy oracle on identical bf16 inputs.

Tolerance (north star): max-abs <= 2e-2 on outputs and gradients against the
float64 oracle fed the same bf16-rounded inputs; gradients come back fp32.
"""

import numpy as np
import pytest
import torch

from conftest import bf16_round, make_batch
from oracle import scfa_oracle as orc

import paper_2306_01160_b200 as scfa

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _np(x):
    return x.detach().float().cpu().numpy().astype(np.float64)


def _check(name, got, want, tol=TOL):
    err = float(np.max(np.abs(got - want))) if want.size else 0.0
    assert np.isfinite(got).all(), f"{name}: non-finite values"
    assert err <= tol, f"{name}: max-abs {err:.3e} > {tol}"


@pytest.mark.parametrize("T", [128, 200, 384])
def test_dense_forward_backward(T):
    B, H, D = 1, 2, 64
    q, k, v = make_batch(B, H, T, D, seed=1)
    dO = bf16_round(np.random.default_rng(3).standard_normal((B, H, T, D)))
    vis = orc.visibility(np.arange(T), np.arange(T))
    O, M, L = orc.attention(q, k, v, vis)
    dq, dk, dv = orc.attention_grads(q, k, v, vis, dO)
    out = scfa.flash_forward(_t(q), _t(k), _t(v))
    _check("O", _np(out.O), O)
    _check("M", _np(out.M), M, 1e-3)
    np.testing.assert_allclose(_np(out.L), L, rtol=2e-2)
    gq, gk, gv = scfa.flash_backward(_t(q), _t(k), _t(v), out, _t(dO))
    _check("dQ", _np(gq), dq)
    _check("dK", _np(gk), dk)
    _check("dV", _np(gv), dv)
    assert out.tiles_computed == scfa.dense_tile_count(T) * B * H


@pytest.mark.parametrize("rt", [False, True], ids=["tiled", "rowtables"])
@pytest.mark.parametrize("T,drop", [(256, 0.5), (1024, 0.5), (300, 0.9), (200, 0.0)])
def test_qk_end_to_end(T, drop, rt):
    B, H, D = 2, 2, 64
    qb, kb, vb = (np.swapaxes(x, 1, 2) for x in make_batch(B, H, T, D, seed=5))
    qk = scfa.random_keep(B, T, H, drop, 11)
    kk = scfa.random_keep(B, T, H, drop, 12)
    dO = bf16_round(np.random.default_rng(4).standard_normal((B, T, H, D)))
    vis = orc.visibility(np.arange(T), np.arange(T))[None, None] & (qk.transpose(0, 2, 1)[..., :, None] > 0) & (
        kk.transpose(0, 2, 1)[..., None, :] > 0)
    eng = lambda x: np.swapaxes(x, 1, 2)
    O, _, _ = orc.attention(eng(qb), eng(kb), eng(vb), vis)
    O = O * (qk.transpose(0, 2, 1)[..., None] > 0)
    dq, dk, dv = orc.attention_grads(eng(qb), eng(kb), eng(vb), vis, eng(dO))
    dq = dq * (qk.transpose(0, 2, 1)[..., None] > 0)
    dk = dk * (kk.transpose(0, 2, 1)[..., None] > 0)
    dv = dv * (kk.transpose(0, 2, 1)[..., None] > 0)
    o = scfa.qk_sparse_attention(_t(qb), _t(kb), _t(vb), _t(qk), _t(kk))
    _check("O", _np(o), eng(O))
    o2, gq, gk, gv = scfa.qk_sparse_attention_fwd_bwd(_t(qb), _t(kb), _t(vb), _t(qk), _t(kk), _t(dO), row_tables=rt)
    _check("O2", _np(o2), eng(O))
    _check("dQ", _np(gq), eng(dq))
    _check("dK", _np(gk), eng(dk))
    _check("dV", _np(gv), eng(dv))


@pytest.mark.parametrize("rt", [False, True], ids=["tiled", "rowtables"])
@pytest.mark.parametrize("T,nb", [(256, 4), (1000, 16), (512, 1)])
def test_hash_end_to_end(T, nb, rt):
    B, H, D = 2, 2, 64
    qb, kb, vb = (np.swapaxes(x, 1, 2) for x in make_batch(B, H, T, D, seed=7))
    hb = scfa.random_buckets(B, T, H, nb, 9)
    dO = bf16_round(np.random.default_rng(5).standard_normal((B, T, H, D)))
    eng = lambda x: np.swapaxes(x, 1, 2)
    hh = hb.transpose(0, 2, 1)
    pos = np.arange(T)
    vis = orc.visibility(pos, pos, hh, hh, exclude_self=True)
    O, _, _ = orc.attention(eng(qb), eng(kb), eng(vb), vis)
    dq, dk, dv = orc.attention_grads(eng(qb), eng(kb), eng(vb), vis, eng(dO))
    ht = _t(hb)
    o = scfa.hash_sparse_attention(_t(qb), _t(kb), _t(vb), ht, ht)
    _check("O", _np(o), eng(O))
    o2, gq, gk, gv = scfa.hash_sparse_attention_fwd_bwd(_t(qb), _t(kb), _t(vb), ht, ht, _t(dO), row_tables=rt)
    _check("O2", _np(o2), eng(O))
    _check("dQ", _np(gq), eng(dq))
    _check("dK", _np(gk), eng(dk))
    _check("dV", _np(gv), eng(dv))


def test_hash_host_streaming_matches_device():
    """Host inputs: per-batch streamed fwd+bwd equals the single device call bit for bit."""
    B, H, T, D, nb = 3, 2, 640, 64, 8
    rng = np.random.default_rng(21)
    x = [torch.from_numpy(rng.standard_normal((B, T, H, D)).astype(np.float32)).to(torch.bfloat16) for _ in range(4)]
    h = torch.from_numpy(scfa.random_buckets(B, T, H, nb, 3))
    dev = [t.cuda() for t in x]
    want = scfa.hash_sparse_attention_fwd_bwd(dev[0], dev[1], dev[2], h.cuda(), h.cuda(), dev[3])
    host = [t.pin_memory() for t in x]
    got = scfa.hash_sparse_attention_fwd_bwd(host[0], host[1], host[2], h, h, host[3])
    torch.cuda.synchronize()
    for a, b in zip(got, want):
        assert not a.is_cuda
        assert torch.equal(a, b.cpu())


@pytest.mark.parametrize("D,pinned", [(48, True), (64, False)])
def test_hash_host_streaming_out_buffers(D, pinned):
    """Host inputs with caller-given result buffers (`out=`, the bench's e2e call), padded
    head dims and pageable memory: the same bits as the device call, in the caller's buffers."""
    B, H, T, nb = 2, 3, 520, 4
    rng = np.random.default_rng(22)
    x = [torch.from_numpy(rng.standard_normal((B, T, H, D)).astype(np.float32)).to(torch.bfloat16) for _ in range(4)]
    h = torch.from_numpy(scfa.random_buckets(B, T, H, nb, 4))
    dev = [t.cuda() for t in x]
    want = scfa.hash_sparse_attention_fwd_bwd(dev[0], dev[1], dev[2], h.cuda(), h.cuda(), dev[3])
    host = [t.pin_memory() for t in x] if pinned else x
    out = [torch.full(w.shape, float("nan"), dtype=w.dtype, pin_memory=pinned) for w in want]
    got = scfa.hash_sparse_attention_fwd_bwd(host[0], host[1], host[2], h, h, host[3], out=out)
    torch.cuda.synchronize()
    for a, o, b in zip(got, out, want):
        assert a.data_ptr() == o.data_ptr()
        assert a.shape == (B, T, H, D)
        assert torch.equal(a, b.cpu())


@pytest.mark.parametrize("fp32,distinct", [(True, False), (False, True), (True, True)])
def test_hash_host_streaming_q_uploaded_last(fp32, distinct):
    """The host-buffer call uploads Q after the ids, K and V and lets the preparation run
    under Q's upload: the paths that read Q before the forward (fp32 inputs converted by
    as_operand; separate query / key ids, where Q is copied into bucket order on the side
    stream) must wait for it.  Sized so Q's upload outlasts the preparation."""
    B, H, T, D, nb = 2, 12, 4096, 64, 16
    rng = np.random.default_rng(23)
    dt = torch.float32 if fp32 else torch.bfloat16
    x = [torch.from_numpy(rng.standard_normal((B, T, H, D)).astype(np.float32)).to(torch.bfloat16).to(dt)
         for _ in range(4)]
    hq = torch.from_numpy(scfa.random_buckets(B, T, H, nb, 5))
    hk = torch.from_numpy(scfa.random_buckets(B, T, H, nb, 6)) if distinct else hq
    dev = [t.cuda() for t in x]
    want = scfa.hash_sparse_attention_fwd_bwd(dev[0], dev[1], dev[2], hq.cuda(), hk.cuda() if distinct else hq.cuda(),
                                              dev[3])
    host = [t.pin_memory() for t in x]
    got = scfa.hash_sparse_attention_fwd_bwd(host[0], host[1], host[2], hq, hk, host[3])
    torch.cuda.synchronize()
    for a, b in zip(got, want):
        assert not a.is_cuda
        assert torch.equal(a, b.cpu())


@pytest.mark.parametrize("mode", ["hash", "qk"])
def test_autograd_matches_fused_fwd_bwd(mode):
    """dynamic_sparse_attention under autograd: same O and gradients as the *_fwd_bwd calls."""
    B, H, T, D = 2, 2, 384, 64
    rng = np.random.default_rng(8)
    x = [torch.from_numpy(rng.standard_normal((B, T, H, D)).astype(np.float32)).to(torch.bfloat16).cuda()
         for _ in range(4)]
    if mode == "hash":
        idx = torch.from_numpy(scfa.random_buckets(B, T, H, 8, 4)).cuda()
        o2, gq, gk, gv = scfa.hash_sparse_attention_fwd_bwd(x[0], x[1], x[2], idx, idx, x[3])
        qi = ki = idx
    else:
        qi = torch.from_numpy(scfa.random_keep(B, T, H, 0.5, 4)).cuda()
        ki = torch.from_numpy(scfa.random_keep(B, T, H, 0.5, 5)).cuda()
        o2, gq, gk, gv = scfa.qk_sparse_attention_fwd_bwd(x[0], x[1], x[2], qi, ki, x[3])
    q, k, v = (t.float().requires_grad_(True) for t in x[:3])
    o = scfa.dynamic_sparse_attention(q, k, v, qi, ki, sparsity_mode=mode)
    o.backward(x[3].float())
    assert torch.equal(o.detach().to(torch.bfloat16), o2)
    for name, a, b in (("dQ", q.grad, gq), ("dK", k.grad, gk), ("dV", v.grad, gv)):
        assert torch.equal(a, b), name


def _hash_oracle(qb, kb, vb, dO, hq, hk, excl):
    eng = lambda x: np.swapaxes(x, 1, 2)
    T_Q, T_KV = qb.shape[1], kb.shape[1]
    vis = orc.visibility(np.arange(T_Q), np.arange(T_KV), hq.transpose(0, 2, 1), hk.transpose(0, 2, 1),
                         exclude_self=excl)
    O, _, _ = orc.attention(eng(qb), eng(kb), eng(vb), vis)
    dq, dk, dv = orc.attention_grads(eng(qb), eng(kb), eng(vb), vis, eng(dO))
    return [eng(x) for x in (O, dq, dk, dv)]


@pytest.mark.parametrize("T", [1, 2, 127, 129])
@pytest.mark.parametrize("excl", [True, False])
def test_hash_fwd_bwd_tiny_and_ragged_lengths(T, excl):
    B, H, D = 2, 3, 64
    qb, kb, vb = (np.swapaxes(x, 1, 2) for x in make_batch(B, H, T, D, seed=51))
    dO = bf16_round(np.random.default_rng(52).standard_normal((B, T, H, D)))
    hb = scfa.random_buckets(B, T, H, 3, 53)
    want = _hash_oracle(qb, kb, vb, dO, hb, hb, excl)
    got = scfa.hash_sparse_attention_fwd_bwd(_t(qb), _t(kb), _t(vb), _t(hb), _t(hb), _t(dO), exclude_self=excl)
    for name, g, w in zip(("O", "dQ", "dK", "dV"), got, want):
        _check(name, _np(g), w)


def test_hash_fwd_bwd_distinct_query_and_key_ids():
    """Separate query / key bucket ids (the general sort path, not the shared fast path)."""
    B, H, T, D = 1, 2, 300, 64
    qb, kb, vb = (np.swapaxes(x, 1, 2) for x in make_batch(B, H, T, D, seed=54))
    dO = bf16_round(np.random.default_rng(55).standard_normal((B, T, H, D)))
    hq = scfa.random_buckets(B, T, H, 4, 56)
    hk = scfa.random_buckets(B, T, H, 4, 57)
    want = _hash_oracle(qb, kb, vb, dO, hq, hk, False)
    got = scfa.hash_sparse_attention_fwd_bwd(_t(qb), _t(kb), _t(vb), _t(hq), _t(hk), _t(dO), exclude_self=False)
    for name, g, w in zip(("O", "dQ", "dK", "dV"), got, want):
        _check(name, _np(g), w)


@pytest.mark.parametrize("T", [1, 2, 129])
def test_qk_fwd_bwd_tiny_and_ragged_lengths(T):
    B, H, D = 2, 2, 64
    qb, kb, vb = (np.swapaxes(x, 1, 2) for x in make_batch(B, H, T, D, seed=58))
    dO = bf16_round(np.random.default_rng(59).standard_normal((B, T, H, D)))
    qk = scfa.random_keep(B, T, H, 0.4, 60)
    kk = scfa.random_keep(B, T, H, 0.4, 61)
    eng = lambda x: np.swapaxes(x, 1, 2)
    pos = np.arange(T)
    vis = orc.visibility(pos, pos) & (qk.transpose(0, 2, 1)[..., :, None] > 0) & (kk.transpose(0, 2, 1)[..., None, :] > 0)
    O, _, _ = orc.attention(eng(qb), eng(kb), eng(vb), vis)
    dq, dk, dv = orc.attention_grads(eng(qb), eng(kb), eng(vb), vis, eng(dO))
    # dropped queries: zero output / gradient; dropped keys: zero dK / dV
    got = scfa.qk_sparse_attention_fwd_bwd(_t(qb), _t(kb), _t(vb), qk, kk, _t(dO))
    for name, g, w in zip(("O", "dQ", "dK", "dV"), got, (O, dq, dk, dv)):
        _check(name, _np(g), eng(w))


def _torch_masked_reference(q, k, v, dO, vis):
    """fp32 torch attention + gradients for one head: q, k, v, dO (T, D); vis (T, T) bool."""
    q, k, v = (x.float().requires_grad_() for x in (q, k, v))
    s = (q @ k.T) / q.shape[-1] ** 0.5
    s = s.masked_fill(~vis, float("-inf"))
    p = torch.softmax(s, dim=-1).nan_to_num(0.0)
    o = p @ v
    o.backward(dO.float())
    return o.detach(), q.grad, k.grad, v.grad


def test_hash_full_cfg2_size_against_torch_fp32():
    """BASELINE configs[1] at full size (B=4 H=12 T=8192 D=64, 16 buckets): the fused
    fwd+bwd against an fp32 torch reference on a sample of heads (same bf16 inputs)."""
    B, H, T, D, nb = 4, 12, 8192, 64, 16
    g = torch.Generator(device="cuda").manual_seed(123)
    q, k, v, dO = (torch.randn((B, T, H, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    ids = torch.randint(0, nb, (B, T, H), device="cuda", generator=g)
    o, dq, dk, dv = scfa.hash_sparse_attention_fwd_bwd(q, k, v, ids, ids, dO)
    pos = torch.arange(T, device="cuda")
    causal = pos[:, None] > pos[None, :]  # exclude_self
    for b, h in ((0, 0), (1, 5), (3, 11)):
        same = ids[b, :, h][:, None] == ids[b, :, h][None, :]
        want = _torch_masked_reference(q[b, :, h], k[b, :, h], v[b, :, h], dO[b, :, h], causal & same)
        for name, got, w in zip(("O", "dQ", "dK", "dV"), (o[b, :, h], dq[b, :, h], dk[b, :, h], dv[b, :, h]), want):
            err = float((got.float() - w).abs().max())
            assert err <= TOL, f"{name} (b={b}, h={h}): max-abs {err:.3e}"


def test_qk_full_cfg3_size_against_torch_fp32():
    """BASELINE configs[2] at full size (B=4 H=12 T=16384 D=64, half of the queries and keys
    dropped): the fused fwd+bwd against an fp32 torch reference on a sample of heads."""
    B, H, T, D = 4, 12, 16384, 64
    g = torch.Generator(device="cuda").manual_seed(321)
    q, k, v, dO = (torch.randn((B, T, H, D), device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    qk = torch.from_numpy(scfa.random_keep(B, T, H, 0.5, 6)).cuda()
    kk = torch.from_numpy(scfa.random_keep(B, T, H, 0.5, 7)).cuda()
    o, dq, dk, dv = scfa.qk_sparse_attention_fwd_bwd(q, k, v, qk, kk, dO)
    pos = torch.arange(T, device="cuda")
    causal = pos[:, None] >= pos[None, :]
    for b, h in ((0, 3), (2, 9)):
        vis = causal & (qk[b, :, h] > 0)[:, None] & (kk[b, :, h] > 0)[None, :]
        want = _torch_masked_reference(q[b, :, h], k[b, :, h], v[b, :, h], dO[b, :, h], vis)
        for name, got, w in zip(("O", "dQ", "dK", "dV"), (o[b, :, h], dq[b, :, h], dk[b, :, h], dv[b, :, h]), want):
            err = float((got.float() - w).abs().max())
            assert err <= TOL, f"{name} (b={b}, h={h}): max-abs {err:.3e}"

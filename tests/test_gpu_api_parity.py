"""Reference-named API calls the golden/end-to-end tests do not reach, checked against
the reference's golden vectors (tests/golden/, written by running the reference):

* kernel-level backward: hash_backward_kernel (hash_sparse.py:182-213) and
  qk_backward_kernel with drops (qk_sparse.py:151-183), composed as the reference
  composes them (dO routed into kernel order, gradients routed back);
* the per-block schedule arrays causal_j_stops / hash_tile_ranges (_kernel.py:45-79)
  element for element against the golden j_start / j_stop;
* compact (with and without index=) and pad_index (qk_sparse.py:41-83);
* dynamic_sparse_attention forward in both modes and its ParameterError (__init__.py:76-90);
* the padding-safety fuzz (test_qk.py:362-392): +-1e8 in the pad rows of compacted
  operands leaves O and every kept row's gradient bitwise unchanged.
"""

import numpy as np
import pytest
import torch

import golden_cases as gc

import paper_2306_01160_b200 as scfa
from paper_2306_01160_b200.tensors import random_tensor_np

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _t(x, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return t if dtype is None else t.to(dtype)


def _np(x):
    return x.detach().to(torch.float64).cpu().numpy()


def _close(label, got, want, tol=TOL):
    assert np.isfinite(got).all(), f"{label}: non-finite values"
    err = float(np.max(np.abs(got - want))) if want.size else 0.0
    assert err <= tol, f"{label}: max-abs {err:.3e} > {tol}"


def _gather_rows(x_bhtd, idx_bht):
    """x (B, H, T, D) rows in idx order along T -> (B, H, T_idx, D)."""
    i = idx_bht.long().clamp(min=0, max=x_bhtd.shape[2] - 1)
    return torch.gather(x_bhtd, 2, i[..., None].expand(*i.shape, x_bhtd.shape[3]))


def _scatter_rows(g_bhtd, idx_bht, T):
    """Inverse of _gather_rows into zeros (B, T, H, D): slots whose index is outside [0, T)
    (pads) are dropped."""
    B, H, Tc, D = g_bhtd.shape
    out = torch.zeros((B, H, T, D), dtype=g_bhtd.dtype, device=g_bhtd.device)
    for b in range(B):
        for h in range(H):
            ix = idx_bht[b, h].long()
            ok = (ix >= 0) & (ix < T)
            out[b, h, ix[ok]] = g_bhtd[b, h][ok]
    return out.transpose(1, 2)


# ------------------------------------------------------------------ kernel-level backward

@pytest.mark.parametrize("name", gc.case_names("hash"))
def test_hash_backward_kernel_golden(name):
    """sort_by_bucket -> hash_forward_kernel -> hash_backward_kernel(dO in sorted order)
    -> inverse permutation, the reference's composition."""
    meta, g = gc.load(name)
    q, k, v, dO = (_t(x, torch.bfloat16) for x in gc.inputs(meta))
    qh, kh = (_t(x) for x in gc.sparsity(meta))
    if meta["shared"]:
        kh = qh
    excl = meta["exclude_self"]
    sb = scfa.sort_by_bucket(scfa.to_heads(q), scfa.to_heads(k), scfa.to_heads(v), scfa.to_heads(qh),
                             scfa.to_heads(kh))
    out = scfa.hash_forward_kernel(sb, exclude_self=excl)
    do_sorted = _gather_rows(scfa.to_heads(dO), sb.q_idx)
    dq_s, dk_s, dv_s = scfa.hash_backward_kernel(sb, out, do_sorted, exclude_self=excl)
    assert dq_s.dtype == torch.float32 and tuple(dq_s.shape) == tuple(sb.q.shape)
    _close("dq", _np(_scatter_rows(dq_s, sb.q_idx, meta["T_Q"])), g["dq"])
    _close("dk", _np(_scatter_rows(dk_s, sb.k_idx, meta["T_KV"])), g["dk"])
    _close("dv", _np(_scatter_rows(dv_s, sb.k_idx, meta["T_KV"])), g["dv"])


@pytest.mark.parametrize("name", gc.case_names("qk"))
def test_qk_backward_kernel_golden(name):
    """qk_preprocess -> qk_forward_kernel -> qk_backward_kernel(dO gathered by
    scatter_index) -> scatter back (dropped positions 0), as SURVEY §8c composes it."""
    meta, g = gc.load(name)
    q, k, v, dO = (_t(x, torch.bfloat16) for x in gc.inputs(meta))
    qk, kk = (_t(x) for x in gc.sparsity(meta))
    prep = scfa.qk_preprocess(q, k, v, qk, kk)
    out = scfa.qk_forward_kernel(prep.q_c, prep.k_c, prep.v_c, prep.q_idx, prep.k_idx)
    # every slot, pads included, gathers a real dO row (scatter_index is unpadded)
    do_c = _gather_rows(scfa.to_heads(dO), prep.scatter_index.transpose(1, 2))
    dq_c, dk_c, dv_c = scfa.qk_backward_kernel(prep.q_c, prep.k_c, prep.v_c, out, do_c, prep.q_idx, prep.k_idx)
    # pad rows of the compacted gradients are exactly zero (qk_sparse.py:176-183)
    qpad = (prep.q_idx == scfa.QUERY_PAD)
    kpad = (prep.k_idx == scfa.KEY_PAD)
    assert not bool(dq_c[qpad].any()) and not bool(dk_c[kpad].any()) and not bool(dv_c[kpad].any())
    _close("dq", _np(_scatter_rows(dq_c, prep.q_idx, meta["T_Q"])), g["dq"])
    _close("dk", _np(_scatter_rows(dk_c, prep.k_idx, meta["T_KV"])), g["dk"])
    _close("dv", _np(_scatter_rows(dv_c, prep.k_idx, meta["T_KV"])), g["dv"])


# ------------------------------------------------------------------ schedule arrays

@pytest.mark.parametrize("name", gc.case_names("qk"))
def test_causal_j_stops_arrays_golden(name):
    meta, g = gc.load(name)
    q, k, v, _ = (_t(x, torch.bfloat16) for x in gc.inputs(meta))
    qk, kk = (_t(x) for x in gc.sparsity(meta))
    prep = scfa.qk_preprocess(q, k, v, qk, kk)
    B, H = meta["B"], meta["H"]
    for b in range(B):
        for h in range(H):
            got = scfa.causal_j_stops(prep.q_idx[b, h], prep.k_idx[b, h])
            np.testing.assert_array_equal(got.cpu().numpy(), g["j_stop"][b, h], err_msg=f"(b={b}, h={h})")
            got2 = scfa.qk_tile_schedule(prep.q_idx[b, h], prep.k_idx[b, h])
            np.testing.assert_array_equal(got2.cpu().numpy(), g["j_stop"][b, h])


@pytest.mark.parametrize("name", gc.case_names("hash"))
def test_hash_tile_ranges_arrays_golden(name):
    meta, g = gc.load(name)
    B, H = meta["B"], meta["H"]
    for b in range(B):
        for h in range(H):
            js, je = scfa.hash_tile_ranges(_t(g["q_hash_sorted"][b, h]), _t(g["q_idx"][b, h]),
                                           _t(g["k_hash_sorted"][b, h]), _t(g["k_idx"][b, h]))
            np.testing.assert_array_equal(js.cpu().numpy(), g["j_start"][b, h], err_msg=f"j_start (b={b}, h={h})")
            np.testing.assert_array_equal(je.cpu().numpy(), g["j_stop"][b, h], err_msg=f"j_stop (b={b}, h={h})")


# ------------------------------------------------------------------ compact / pad_index

@pytest.mark.parametrize("name", gc.case_names("qk"))
def test_compact_and_pad_index_golden(name):
    meta, g = gc.load(name)
    q, k, v, _ = (_t(x, torch.bfloat16) for x in gc.inputs(meta))
    qk, kk = (_t(x) for x in gc.sparsity(meta))
    cq = scfa.compact(qk, q)
    np.testing.assert_array_equal(cq.index.cpu().numpy(), g["q_index"])
    np.testing.assert_array_equal(cq.indices_per_head.cpu().numpy(), g["q_counts"])
    ck = scfa.compact(kk, k)
    np.testing.assert_array_equal(ck.index.cpu().numpy(), g["k_index"])
    np.testing.assert_array_equal(ck.indices_per_head.cpu().numpy(), g["k_counts"])
    # rows are the input rows at the index (a pure gather: bitwise)
    want = torch.gather(q, 1, cq.index.long()[..., None].expand(*cq.index.shape, q.shape[3]))
    assert torch.equal(cq.compact, want)
    # index= reuses K's index for V (qk_sparse.py:61-66); no counts come back
    cv = scfa.compact(kk, v, index=ck.index)
    assert cv.indices_per_head is None
    assert torch.equal(cv.compact, torch.gather(v, 1, ck.index.long()[..., None].expand(*ck.index.shape, v.shape[3])))
    # pad_index: the padded (B, H, T_c) vectors of the golden case, transposed
    pq = scfa.pad_index(cq.index, cq.indices_per_head, scfa.QUERY_PAD)
    pk = scfa.pad_index(ck.index, ck.indices_per_head, scfa.KEY_PAD)
    np.testing.assert_array_equal(pq.transpose(1, 2).cpu().numpy(), g["q_idx"])
    np.testing.assert_array_equal(pk.transpose(1, 2).cpu().numpy(), g["k_idx"])
    assert pq.data_ptr() != cq.index.data_ptr()  # a copy (qk_sparse.py:80)


def test_compact_rejects_bad_keep_and_index():
    x = torch.randn((1, 8, 2, 64), device="cuda").to(torch.bfloat16)
    keep = torch.ones((1, 8, 2), device="cuda")
    keep[0, 3, 1] = 0.5
    with pytest.raises(scfa.ShapeError):
        scfa.compact(keep, x)
    with pytest.raises(scfa.ShapeError):
        scfa.compact(None, x, index=torch.full((1, 4, 2), 8, device="cuda"))


# ------------------------------------------------------------------ router

@pytest.mark.parametrize("name", ["hash_small", "hash_self", "qk_small", "qk_cfg1"])
def test_dynamic_sparse_attention_forward_golden(name):
    meta, g = gc.load(name)
    q, k, v, _ = (_t(x, torch.bfloat16) for x in gc.inputs(meta))
    a, b = (_t(x) for x in gc.sparsity(meta))
    if meta["kind"] == "hash":
        if not meta["exclude_self"]:
            pytest.skip("the router keeps the reference default exclude_self=True")
        o = scfa.dynamic_sparse_attention(q, k, v, a, a if meta["shared"] else b, sparsity_mode="hash")
    else:
        o = scfa.dynamic_sparse_attention(q, k, v, a, b, sparsity_mode="qk")
    _close("O", _np(o), g["O"])


def test_dynamic_sparse_attention_scale_and_bad_mode():
    meta, g = gc.load("hash_small")
    q, k, v, _ = (_t(x, torch.bfloat16) for x in gc.inputs(meta))
    a, _ = (_t(x) for x in gc.sparsity(meta))
    d = meta["D"]
    o1 = scfa.dynamic_sparse_attention(q, k, v, a, a)  # default mode is "hash"
    o2 = scfa.dynamic_sparse_attention(q, k, v, a, a, sm_scale=1.0 / d ** 0.5)
    assert torch.equal(o1, o2)
    with pytest.raises(scfa.ParameterError):
        scfa.dynamic_sparse_attention(q, k, v, a, a, sparsity_mode="dense")


# ------------------------------------------------------------------ padding safety

@pytest.mark.parametrize("B,H,T,D", [(1, 2, 24, 3), (2, 3, 300, 64), (1, 2, 260, 128)])
def test_padding_safety_fuzz_bitwise(B, H, T, D):
    """test_qk.py:362-392: pad rows of the compacted operands filled with +-1e8 change
    neither O nor any kept row's gradient, bitwise."""
    bf = lambda x: _t(gc.bf16(x), torch.bfloat16)
    q, k, v = (bf(np.swapaxes(random_tensor_np((B, H, T, D), 45 + i), 1, 2)) for i in range(3))
    keep_q = scfa.random_keep(B, T, H, 0.4, 46)
    keep_k = scfa.random_keep(B, T, H, 0.4, 47)
    prep = scfa.qk_preprocess(q, k, v, keep_q, keep_k)
    out = scfa.qk_forward_kernel(prep.q_c, prep.k_c, prep.v_c, prep.q_idx, prep.k_idx)
    d_out = bf(random_tensor_np(tuple(prep.q_c.shape), 48))
    grads = scfa.qk_backward_kernel(prep.q_c, prep.k_c, prep.v_c, out, d_out, prep.q_idx, prep.k_idx)

    rng = np.random.default_rng(49)
    q_f, k_f, v_f = prep.q_c.clone(), prep.k_c.clone(), prep.v_c.clone()
    q_pads = prep.q_idx == scfa.QUERY_PAD
    k_pads = prep.k_idx == scfa.KEY_PAD
    for x, pads in ((q_f, q_pads), (k_f, k_pads), (v_f, k_pads)):
        n = int(pads.sum())
        x[pads] = _t(rng.uniform(-1e8, 1e8, size=(n, D)), torch.bfloat16)
    assert int(q_pads.sum()) > 0 and int(k_pads.sum()) > 0
    fuzzed = scfa.qk_forward_kernel(q_f, k_f, v_f, prep.q_idx, prep.k_idx)
    assert torch.equal(fuzzed.O, out.O)
    fg = scfa.qk_backward_kernel(q_f, k_f, v_f, fuzzed, d_out, prep.q_idx, prep.k_idx)
    kept_q, kept_k = ~q_pads, ~k_pads
    assert torch.equal(fg[0][kept_q], grads[0][kept_q])
    assert torch.equal(fg[1][kept_k], grads[1][kept_k])
    assert torch.equal(fg[2][kept_k], grads[2][kept_k])


# ------------------------------------------------------------------ single-pass backward

@pytest.mark.parametrize("name", [n for n in gc.case_names("hash")])
def test_single_pass_backward_golden(name):
    """scfa_attn_bwd (dQ, dK, dV in one key-stationary sweep, dQ reduced in fp32) against the
    reference goldens; cases it does not cover (distinct ids, D = 128) fall back to the
    two-pass backward and must match just the same."""
    meta, g = gc.load(name)
    q, k, v, dO = (_t(x, torch.bfloat16) for x in gc.inputs(meta))
    qh, kh = (_t(x) for x in gc.sparsity(meta))
    if meta["shared"]:
        kh = qh
    o, dq, dk, dv = scfa.hash_sparse_attention_fwd_bwd(q, k, v, qh, kh, dO, exclude_self=meta["exclude_self"],
                                                       single_pass=True)
    _close("O", _np(o), g["O"])
    for label, got in (("dq", dq), ("dk", dk), ("dv", dv)):
        _close(label, _np(got), g[label])


@pytest.mark.parametrize("B,T,H,nb", [(1, 300, 2, 4), (4, 8192, 12, 16), (2, 16384, 3, 64)])
def test_single_pass_matches_two_pass(B, T, H, nb):
    """dK / dV bit for bit (same arithmetic and order); dQ to fp32 reduction-order noise."""
    g = torch.Generator(device="cuda").manual_seed(T + nb)
    q, k, v, dO = (torch.randn((B, T, H, 64), device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    ids = torch.randint(0, nb, (B, T, H), device="cuda", generator=g)
    a = scfa.hash_sparse_attention_fwd_bwd(q, k, v, ids, ids, dO, single_pass=True)
    b = scfa.hash_sparse_attention_fwd_bwd(q, k, v, ids, ids, dO)
    assert torch.equal(a[0], b[0]) and torch.equal(a[2], b[2]) and torch.equal(a[3], b[3])
    err = float((a[1] - b[1]).abs().max())
    assert err <= 1e-4 * max(1.0, float(b[1].abs().max())), err

"""GPU schedule parity: the visibility runs and exact tile lists of scfa_build_schedule
against a brute-force visibility matrix built by the oracle on the same sorted /
compacted index vectors (_tile_mask semantics, _kernel.py:82-89).

Bars (bit-exact): every row's run [lo, hi) is exactly its set of visible slots; a tile
is listed iff it holds a visible pair, flagged full iff all its pairs are visible;
the listed-tile totals match.
"""

import numpy as np
import pytest
import torch

from oracle import scfa_oracle as orc

import paper_2306_01160_b200 as scfa
from paper_2306_01160_b200 import hash_sparse as hs

pytestmark = pytest.mark.gpu


def _check_problem(prob, vis):
    """vis: (BH, T_q, T_kv) bool in kernel slot order."""
    sched = prob.schedule("fwd", "dq", "dkdv")
    BH, Tq, Tk = vis.shape
    qr = sched["q_runs"].cpu().numpy()
    kr = sched["k_runs"].cpu().numpy()
    for bh in range(BH):
        for s in range(prob.Tq_pad):
            want = np.zeros(Tk, bool) if s >= Tq else vis[bh, s]
            got = np.zeros(Tk, bool)
            got[qr[bh, s, 0]:qr[bh, s, 1]] = True
            assert np.array_equal(got, want), f"q run bh={bh} slot={s}: {qr[bh, s]}"
        for s in range(prob.Tkv_pad):
            want = np.zeros(Tq, bool) if s >= Tk else vis[bh, :, s]
            got = np.zeros(Tq, bool)
            got[kr[bh, s, 0]:kr[bh, s, 1]] = True
            assert np.array_equal(got, want), f"k run bh={bh} slot={s}: {kr[bh, s]}"
    totals = prob._tiles_total.cpu().numpy()
    for slot, (name, rows_q, cb) in enumerate((("fwd", True, 128), ("dq", True, 64), ("dkdv", False, 64))):
        lst, cnt, _ = sched[name]
        lst = lst.cpu().numpy().view(np.uint16)
        cnt = cnt.cpu().numpy()
        v = vis if rows_q else np.swapaxes(vis, 1, 2)
        n_rb = -(-v.shape[1] // 128)
        n_cb = -(-v.shape[2] // cb)
        total = 0
        for bh in range(BH):
            for rb in range(n_rb):
                rows = np.zeros((128, n_cb * cb), bool)
                blk = v[bh, rb * 128:(rb + 1) * 128]
                rows[:blk.shape[0], :blk.shape[1]] = blk
                tiles = rows.reshape(128, n_cb, cb)
                any_ = tiles.any(axis=(0, 2))
                all_ = tiles.all(axis=(0, 2))
                want = [c | (0x8000 if all_[c] else 0) for c in range(n_cb) if any_[c]]
                got = list(lst[bh, rb, :cnt[bh, rb]])
                assert got == want, f"{name} bh={bh} rb={rb}: {got[:8]} vs {want[:8]}"
                total += len(want)
        assert totals[slot] == total


@pytest.mark.parametrize("T,nb,excl,seed", [(300, 4, True, 0), (1024, 16, True, 1), (512, 1, False, 2),
                                            (700, 64, True, 3)])
def test_hash_runs_and_lists(T, nb, excl, seed):
    B, H, D = 1, 2, 64
    dev = torch.device("cuda")
    x = torch.zeros((B, T, H, D), dtype=torch.bfloat16, device=dev)
    h = torch.from_numpy(scfa.random_buckets(B, T, H, nb, seed)).to(dev)
    sb = hs._sort_batch(x, x, x, h, h, "bthd", exclude_self=excl)
    prob = hs._problem_of(sb, excl)
    qi = sb.q_idx.cpu().numpy().reshape(B * H, T)
    qh = sb.q_hash.cpu().numpy().reshape(B * H, T)
    vis = orc.visibility(qi, qi, qh, qh, exclude_self=excl)
    _check_problem(prob, vis)


def test_hash_rect_runs_and_lists():
    B, H, D, Tq, Tk = 1, 2, 64, 200, 333
    dev = torch.device("cuda")
    xq = torch.zeros((B, Tq, H, D), dtype=torch.bfloat16, device=dev)
    xk = torch.zeros((B, Tk, H, D), dtype=torch.bfloat16, device=dev)
    qh = torch.from_numpy(scfa.random_buckets(B, Tq, H, 8, 5)).to(dev)
    kh = torch.from_numpy(scfa.random_buckets(B, Tk, H, 8, 6)).to(dev)
    sb = hs._sort_batch(xq, xk, xk, qh, kh, "bthd")
    prob = hs._problem_of(sb, True)
    qi = sb.q_idx.cpu().numpy().reshape(B * H, Tq)
    ki = sb.k_idx.cpu().numpy().reshape(B * H, Tk)
    vis = orc.visibility(qi, ki, sb.q_hash.cpu().numpy().reshape(B * H, Tq),
                         sb.k_hash.cpu().numpy().reshape(B * H, Tk), exclude_self=True)
    _check_problem(prob, vis)


@pytest.mark.parametrize("T,drop,seed", [(300, 0.5, 0), (1024, 0.3, 1), (256, 0.0, 2), (400, 0.95, 3)])
def test_qk_runs_and_lists(T, drop, seed):
    B, H, D = 2, 2, 64
    dev = torch.device("cuda")
    x = torch.zeros((B, T, H, D), dtype=torch.bfloat16, device=dev)
    qk = torch.from_numpy(scfa.random_keep(B, T, H, drop, seed)).to(dev)
    kk = torch.from_numpy(scfa.random_keep(B, T, H, drop, seed + 100)).to(dev)
    prep = scfa.qk_preprocess(x, x, x, qk, kk)
    prob = prep.problem
    qi = prep.q_idx.cpu().numpy().reshape(B * H, -1).astype(np.int64)
    ki = prep.k_idx.cpu().numpy().reshape(B * H, -1).astype(np.int64)
    vis = orc.visibility(qi, ki)
    vis &= (qi >= 0)[..., :, None] & (ki < orc.KEY_PAD)[..., None, :]
    _check_problem(prob, vis)


def test_dense_runs_and_lists():
    from paper_2306_01160_b200.dense import causal_problem

    T = 513
    prob = causal_problem(1, 1, T, 64, torch.device("cuda"))
    vis = orc.visibility(np.arange(T), np.arange(T))[None]
    _check_problem(prob, vis)


# T >= 4096 with few slices runs the cluster sort (4 CTAs per slice; nb > 256 its
# multi-pass fallback, nb = 1 the all-zero ids)
@pytest.mark.parametrize("T,nb,excl,seed", [(300, 4, True, 0), (2048, 16, False, 1), (4096, 300, True, 2),
                                            (1000, 1, True, 3), (8192, 16, True, 4), (16384, 64, False, 5),
                                            (4096, 1, True, 6), (5000, 7, True, 7)])
def test_fused_prepare_matches_general_path(T, nb, excl, seed):
    """scfa_hash_prepare (shared ids) == hash_sort + build_aux + runs_kernel, bit for bit."""
    from paper_2306_01160_b200._kernel import Problem

    B, H, D = 2, 3, 64
    dev = torch.device("cuda")
    x = torch.zeros((B, T, H, D), dtype=torch.bfloat16, device=dev)
    h = torch.from_numpy(scfa.random_buckets(B, T, H, nb, seed)).to(dev)
    sb = hs._sort_batch(x, x, x, h, h, "bthd", exclude_self=excl)
    fused = sb.problem
    # reference order: stable argsort of the bucket ids per (b, h)
    want = np.argsort(h.cpu().numpy().transpose(0, 2, 1).reshape(B * H, T), axis=1, kind="stable")
    assert np.array_equal(sb.q_perm.cpu().numpy(), want)
    assert np.array_equal(sb.q_rank.cpu().numpy(), np.argsort(want, axis=1))
    # the sorted vectors and row table the sort writes (itself, on the cluster path)
    T_pad = fused.Tq_pad
    perm = sb.q_perm.cpu().numpy()
    hs_np = h.cpu().numpy().transpose(0, 2, 1).reshape(B * H, T)
    qi, ki = fused.q_idx.cpu().numpy(), fused.k_idx.cpu().numpy()
    qh, kh = fused.q_hash.cpu().numpy(), fused.k_hash.cpu().numpy()
    assert np.array_equal(qi[:, :T], perm) and np.array_equal(ki[:, :T], perm)
    sorted_ids = np.take_along_axis(hs_np, perm, axis=1)
    assert np.array_equal(qh[:, :T], sorted_ids) and np.array_equal(kh[:, :T], sorted_ids)
    assert (qi[:, T:] == -1).all() and (ki[:, T:] == 0x7FFFFFFF).all()
    assert (qh[:, T:] == -3).all() and (kh[:, T:] == -2).all()
    rows = fused.rows.q_rows.cpu().numpy()
    bh = np.arange(B * H)[:, None]
    want_rows = ((bh // H) * T + perm) * H + bh % H
    assert np.array_equal(rows[:, :T], want_rows)
    assert (rows[:, T:] == want_rows[:, :1]).all()
    flags = fused.flags
    general = Problem(B, H, T, T, D, fused.q_idx.clone(), fused.k_idx.clone(), fused.q_hash.clone(),
                      fused.k_hash.clone(), flags=flags)
    g = general.schedule("fwd", "dq", "dkdv")
    f = fused.schedule("fwd", "dq", "dkdv")
    for key in ("q_runs", "k_runs"):
        assert torch.equal(g[key], f[key]), key
    for name in ("fwd", "dq", "dkdv"):
        assert torch.equal(g[name][1], f[name][1]), name

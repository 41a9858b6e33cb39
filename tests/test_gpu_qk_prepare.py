"""GPU parity of the fused QK preparation (scfa_qk_prepare) used by the static-size fused
QK fwd + bwd: every output bit-exact against the multi-pass path it replaces (compaction per
side, aux vectors, row maps, scfa_build_schedule's runs) and against numpy / brute force:

  perm  == argsort(~kept, stable)                      (qk_sparse.py:59)
  idx   == pad_index of the kept prefix                (qk_sparse.py:74-83)
  runs  == the visible slot run of every row            (_tile_mask, _kernel.py:82-89)
  lists == non-empty / full tiles of the visibility     (exact tile lists)
"""

import numpy as np
import pytest
import torch

from oracle import scfa_oracle as orc

import paper_2306_01160_b200 as scfa
from paper_2306_01160_b200 import qk_sparse as qs
from paper_2306_01160_b200.tensors import KEY_PAD, QUERY_PAD

from test_gpu_schedule import _check_problem

pytestmark = pytest.mark.gpu


def _static_pair(B, Tq, Tk, H, qk_np, kk_np, dtype=torch.float64):
    dev = torch.device("cuda")
    q = torch.randn((B, Tq, H, 64), device=dev).to(torch.bfloat16)
    k = torch.randn((B, Tk, H, 64), device=dev).to(torch.bfloat16)
    v = torch.randn((B, Tk, H, 64), device=dev).to(torch.bfloat16)
    qk = torch.from_numpy(qk_np).to(dev, dtype)
    kk = torch.from_numpy(kk_np).to(dev, dtype)
    e1 = torch.zeros(1, dtype=torch.int32, device=dev)
    e2 = torch.zeros(1, dtype=torch.int32, device=dev)
    fused = qs._prepare_static(q, k, v, qk, kk, e1)
    passes = qs._prepare_static_passes(q, k, v, qk, kk, e2)
    torch.cuda.synchronize()
    return fused, passes, (q, k, v), (e1, e2)


CASES = [
    (2, 1024, 1024, 3, 0.5, 0),
    (1, 300, 300, 2, 0.3, 1),      # T not a multiple of 128
    (1, 200, 333, 2, 0.5, 2),      # rectangular T_Q < T_KV
    (1, 333, 200, 2, 0.5, 3),      # rectangular T_Q > T_KV
    (1, 4096, 4096, 2, 0.9, 4),
    (1, 16384, 16384, 1, 0.5, 5),  # the kernel's largest T
]


@pytest.mark.parametrize("B,Tq,Tk,H,drop,seed", CASES)
def test_fused_prepare_matches_passes_and_numpy(B, Tq, Tk, H, drop, seed):
    qk = scfa.random_keep(B, Tq, H, drop, seed)
    kk = scfa.random_keep(B, Tk, H, drop, seed + 100)
    fused, passes, (q, k, v), _ = _static_pair(B, Tq, Tk, H, qk, kk)
    pf, pp = fused.problem, passes.problem
    # perm / rank / padded idx / row tables: bitwise the multi-pass path
    for a, b in ((fused.q_rank, passes.q_rank), (fused.k_rank, passes.k_rank), (pf.q_idx, pp.q_idx),
                 (pf.k_idx, pp.k_idx), (pf.rows.q_rows, pp.rows.q_rows), (pf.rows.k_rows, pp.rows.k_rows),
                 (fused.scatter_index, passes.scatter_index), (fused.k_c, passes.k_c), (fused.v_c, passes.v_c)):
        assert torch.equal(a, b)
    # runs: bitwise what scfa_build_schedule computes from the same index vectors
    sf, sp = pf.schedule("fwd", "dq", "dkdv"), pp.schedule("fwd", "dq", "dkdv")
    for key in ("q_runs", "k_runs"):
        assert torch.equal(sf[key], sp[key]), key
    for name in ("fwd", "dq", "dkdv"):
        lf, cf, _ = sf[name]
        lp, cp, _ = sp[name]
        assert torch.equal(cf, cp), name
        cn, a, b = cf.cpu().numpy(), lf.cpu().numpy(), lp.cpu().numpy()  # entries past the count are unused
        for bh in range(cn.shape[0]):
            for rb in range(cn.shape[1]):
                assert np.array_equal(a[bh, rb, :cn[bh, rb]], b[bh, rb, :cn[bh, rb]]), (name, bh, rb)
    # numpy: perm == argsort(~kept, stable) per head, padded idx
    perm_q = fused.scatter_index.transpose(1, 2).reshape(B * H, Tq).cpu().numpy()
    for b in range(B):
        for h in range(H):
            want = np.argsort(~(qk[b, :, h] == 1), kind="stable")
            assert np.array_equal(perm_q[b * H + h], want)
            n = int((qk[b, :, h] == 1).sum())
            qi = fused.q_idx[b, h].cpu().numpy()
            assert np.array_equal(qi[:n], want[:n]) and (qi[n:] == QUERY_PAD).all()
            nk = int((kk[b, :, h] == 1).sum())
            ki = fused.k_idx[b, h].cpu().numpy()
            assert np.array_equal(ki[:nk], np.flatnonzero(kk[b, :, h] == 1)) and (ki[nk:] == KEY_PAD).all()


@pytest.mark.parametrize("B,Tq,Tk,H,drop,seed", CASES[:4])
def test_fused_prepare_runs_and_lists_brute_force(B, Tq, Tk, H, drop, seed):
    qk = scfa.random_keep(B, Tq, H, drop, seed)
    kk = scfa.random_keep(B, Tk, H, drop, seed + 100)
    fused, _, _, _ = _static_pair(B, Tq, Tk, H, qk, kk)
    qi = fused.q_idx.cpu().numpy().reshape(B * H, -1).astype(np.int64)
    ki = fused.k_idx.cpu().numpy().reshape(B * H, -1).astype(np.int64)
    vis = orc.visibility(qi, ki)
    vis &= (qi >= 0)[..., :, None] & (ki < orc.KEY_PAD)[..., None, :]
    _check_problem(fused.problem, vis)


@pytest.mark.parametrize("kept", [0.0, 1.0])
def test_fused_prepare_all_or_nothing(kept):
    B, T, H = 1, 640, 2
    m = np.full((B, T, H), kept)
    fused, passes, _, _ = _static_pair(B, T, T, H, m, m)
    assert torch.equal(fused.problem.q_idx, passes.problem.q_idx)
    sf, sp = fused.problem.schedule("fwd", "dq", "dkdv"), passes.problem.schedule("fwd", "dq", "dkdv")
    for key in ("q_runs", "k_runs"):
        assert torch.equal(sf[key], sp[key])


@pytest.mark.parametrize("dtype", [torch.float32, torch.uint8, torch.bool])
def test_fused_prepare_keep_dtypes(dtype):
    B, T, H = 1, 500, 2
    qk = scfa.random_keep(B, T, H, 0.5, 11)
    kk = scfa.random_keep(B, T, H, 0.5, 12)
    fused, passes, _, _ = _static_pair(B, T, T, H, qk, kk, dtype)
    assert torch.equal(fused.q_rank, passes.q_rank) and torch.equal(fused.k_rank, passes.k_rank)


def test_fused_prepare_flags_bad_keep():
    B, T, H = 1, 256, 2
    qk = scfa.random_keep(B, T, H, 0.5, 1)
    qk[0, 7, 1] = 0.5
    kk = scfa.random_keep(B, T, H, 0.5, 2)
    _, _, _, (e1, e2) = _static_pair(B, T, T, H, qk, kk)
    assert int(e1.item()) == int(e2.item()) != 0

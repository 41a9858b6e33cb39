"""Hash path step-by-step diagnostics."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
from conftest import bf16_round, make_batch
from oracle import scfa_oracle as orc
import paper_2306_01160_b200 as scfa
from paper_2306_01160_b200 import hash_sparse as hs, _kernel as K, _lib

def P(*a): print(*a, flush=True)
def t(x): return torch.from_numpy(np.ascontiguousarray(x)).cuda()
def n(x): return x.detach().float().cpu().numpy().astype(np.float64)
def S(msg): torch.cuda.synchronize(); P("  ok:", msg)

for (T, nb, excl) in [(256, 4, True), (256, 4, False), (256, 1, False), (1000, 16, True)]:
    P(f"== hash T={T} nb={nb} exclude_self={excl}")
    B, H, D = 2, 2, 64
    qb, kb, vb = (np.swapaxes(x, 1, 2) for x in make_batch(B, H, T, D, seed=7))
    hb = scfa.random_buckets(B, T, H, nb, 9)
    ht = t(hb)
    q, k, v = (K.as_operand(t(x)) for x in (qb, kb, vb))
    sb = hs._sort_batch(q, k, v, ht, ht, "bthd")
    S("sort+gather+aux")
    prob = hs._problem_of(sb, excl)
    for key in [(True, 128), (True, 64), (False, 64)]:
        lst, cnt, stride = prob.tile_list(*key)
        S(f"tile list {key}: counts {cnt.cpu().numpy().ravel()[:8]}")
        c0 = int(cnt[0, 0])
        P("     first list:", (lst[0, 0, :c0].cpu().numpy().astype(np.int64) & 0xFFFF))
    out = K.attention_forward(prob, sb.q, sb.k, sb.v)
    S("fwd")
    hh = hb.transpose(0, 2, 1)
    vis = orc.visibility(np.arange(T), np.arange(T), hh, hh, exclude_self=excl)
    eng = lambda x: np.swapaxes(x, 1, 2)
    O, M, L = orc.attention(eng(qb), eng(kb), eng(vb), vis)
    o = hs._scatter(out.O, sb.q_rank, "bthd")
    P("  O err", np.abs(n(o) - eng(O)).max())
    dO = bf16_round(np.random.default_rng(5).standard_normal((B, T, H, D)))
    d_s = hs._gather(K.as_operand(t(dO)), sb.q_perm, "bthd")
    S("gather dO")
    g = K.attention_backward(prob, sb.q, sb.k, sb.v, out, d_s)
    S("bwd")
    want = orc.attention_grads(eng(qb), eng(kb), eng(vb), vis, eng(dO))
    for nm, a, r, b in zip("QKV", g, (sb.q_rank, sb.k_rank, sb.k_rank), want):
        P(f"  d{nm} err", np.abs(n(hs._scatter(a, r, "bthd")) - eng(b)).max())
P("DIAG2 DONE")

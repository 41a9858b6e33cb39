"""Step-by-step GPU diagnostics (prints as it goes; run under `timeout`)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
from conftest import bf16_round, make_batch
from oracle import scfa_oracle as orc
import paper_2306_01160_b200 as scfa

def P(*a):
    print(*a, flush=True)

def t(x): return torch.from_numpy(np.ascontiguousarray(x)).cuda()
def n(x): return x.detach().float().cpu().numpy().astype(np.float64)

P("device", torch.cuda.get_device_name(0))
# 1. compaction
B, T, H = 2, 300, 3
keep = scfa.random_keep(B, T, H, 0.5, 1)
cr = scfa.compact(t(keep), t(np.zeros((B, T, H, 64), np.float32)))
order, counts = orc.compact_order(keep)
buf = counts.max()
P("compact index ok:", np.array_equal(cr.index.cpu().numpy(), order[:, :buf]), "counts ok:",
  np.array_equal(cr.indices_per_head.cpu().numpy(), counts))
# 2. sort
hb = scfa.random_buckets(B, T, H, 16, 2)
q = np.random.default_rng(0).standard_normal((B, H, T, 64))
sb = scfa.sort_by_bucket(t(q), t(q), t(q), t(hb.transpose(0, 2, 1).copy()), t(hb.transpose(0, 2, 1).copy()))
o_ref = orc.bucket_order(hb.transpose(0, 2, 1))
P("sort ok:", np.array_equal(sb.q_idx.cpu().numpy(), o_ref))
torch.cuda.synchronize()

def dense_case(T, D=64):
    qq, kk, vv = make_batch(1, 2, T, D, seed=1)
    dO = bf16_round(np.random.default_rng(3).standard_normal((1, 2, T, D)))
    vis = orc.visibility(np.arange(T), np.arange(T))
    O, M, L = orc.attention(qq, kk, vv, vis)
    t0 = time.time()
    out = scfa.flash_forward(t(qq), t(kk), t(vv))
    torch.cuda.synchronize()
    P(f"dense T={T} D={D} fwd ran in {time.time()-t0:.2f}s")
    eO = np.abs(n(out.O) - O)
    P("  O max err", eO.max(), "per-128-row-block:", [float(eO[..., i:i+128, :].max()) for i in range(0, T, 128)])
    P("  O sample got", n(out.O)[0, 0, 5, :4], "want", O[0, 0, 5, :4])
    P("  M err", np.abs(n(out.M) - M).max(), "L rel", np.abs(n(out.L) / L - 1).max())
    g = scfa.flash_backward(t(qq), t(kk), t(vv), out, t(dO))
    torch.cuda.synchronize()
    want = orc.attention_grads(qq, kk, vv, vis, dO)
    for nm, a, b in zip("QKV", g, want):
        e = np.abs(n(a) - b)
        P(f"  d{nm} max err", e.max(), "blocks:", [float(e[..., i:i+128, :].max()) for i in range(0, T, 128)])

for T in (128, 256, 200):
    dense_case(T)
dense_case(256, 128)
P("DIAG DONE")

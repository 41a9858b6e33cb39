import sys, torch, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2306_01160_b200 as scfa
from conftest import make_batch, bf16_round
B, H, T, D = 2, 2, 300, 64
x = [np.ascontiguousarray(np.swapaxes(a, 1, 2)) for a in make_batch(B, H, T, D, seed=3)]
dO = bf16_round(np.random.default_rng(4).standard_normal((B, T, H, D)))
h = torch.from_numpy(scfa.random_buckets(B, T, H, 4, 5))
dev = [torch.from_numpy(a).cuda().to(torch.bfloat16) for a in x + [dO]]
for trial in range(3):
    want = scfa.hash_sparse_attention_fwd_bwd(dev[0], dev[1], dev[2], h.cuda(), h.cuda(), dev[3])
    want2 = scfa.hash_sparse_attention_fwd_bwd(dev[0], dev[1], dev[2], h.cuda(), h.cuda(), dev[3])
    host = [t.cpu() for t in dev]
    got = scfa.hash_sparse_attention_fwd_bwd(host[0], host[1], host[2], h, h, host[3])
    torch.cuda.synchronize()
    for name, a, b, c in zip("O dQ dK dV".split(), got, want, want2):
        d = (a.float() - b.cpu().float()).abs().max().item()
        d2 = (c.float() - b.float()).abs().max().item()
        print(trial, name, "host-vs-dev", d, "dev-vs-dev", d2)

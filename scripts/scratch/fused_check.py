import torch, sys, time
sys.path.insert(0, '.')
import paper_2306_01160_b200 as scfa
from paper_2306_01160_b200 import hash_sparse as hs
for (B,T,H,nb) in [(1,256,2,4),(1,1000,2,8),(4,8192,12,16)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    q,k,v,dO = (torch.randn((B,T,H,64), device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    ids = torch.randint(0, nb, (B,T,H), device="cuda", generator=g)
    a = scfa.hash_sparse_attention_fwd_bwd(q,k,v,ids,ids,dO, single_pass=True)
    b = scfa.hash_sparse_attention_fwd_bwd(q,k,v,ids,ids,dO)
    torch.cuda.synchronize()
    print(B,T,H,nb, [float((x.float()-y.float()).abs().max()) for x,y in zip(a,b)], [float(y.abs().max()) for y in b], flush=True)

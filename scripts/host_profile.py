import cProfile, pstats, os, sys, time
import torch
sys.path.insert(0, "/root/repo")
from paper_2306_01160_b200 import hash_sparse as hs
B,T,H,D,nb=4,8192,12,64,16
dev=torch.device("cuda")
g=torch.Generator(device=dev).manual_seed(0)
q,k,v,dO=(torch.randn((B,T,H,D),device=dev,generator=g).to(torch.bfloat16) for _ in range(4))
ids=torch.randint(0,nb,(B,T,H),device=dev,generator=g)
f=lambda: hs._fwd_bwd(q,k,v,ids,ids,dO,exclude_self=True)
for _ in range(5): f()
torch.cuda.synchronize()
t0=time.perf_counter()
for _ in range(50): f()
t1=time.perf_counter()
torch.cuda.synchronize(); t2=time.perf_counter()
print("host ms/call %.3f  (with sync %.3f)"%((t1-t0)/50*1e3,(t2-t0)/50*1e3))
pr=cProfile.Profile(); pr.enable()
for _ in range(50): f()
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

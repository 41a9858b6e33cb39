import torch, sys, os
sys.path.insert(0, os.getcwd())
from paper_2306_01160_b200 import lm
from paper_2306_01160_b200.autograd import hash_sparse_attention_autograd as hsa
torch.manual_seed(0)
B,T,H,D=4,8192,12,64
def timeit(f, n=5):
    for _ in range(2): f()
    torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)/n
q=torch.randn(B,T,H,D,device="cuda",dtype=torch.bfloat16,requires_grad=True)
v=torch.randn(B,T,H,D,device="cuda",dtype=torch.bfloat16,requires_grad=True)
do=torch.randn(B,T,H,D,device="cuda",dtype=torch.bfloat16)
R=torch.randn(H,D,8,device="cuda")
k=torch.nn.functional.normalize(q.detach(),dim=-1).requires_grad_()
ids_lsh=lm.lsh_bucket_ids(k,R)
ids_rand=torch.randint(0,16,(B,T,H),device="cuda")
for name,ids in [("rand",ids_rand),("lsh",ids_lsh)]:
    cnt=torch.stack([(ids==b).sum() for b in range(16)]).float()
    coll=float((cnt**2).sum()/ (B*H) / T**2)
    for ex in (True,False):
        def f():
            o=hsa(q,k,v,ids,ids,exclude_self=ex,check=False); o.backward(do)
        print(name,"excl",ex,"collision frac %.4f"%coll, "ms %.3f"%timeit(f))
# LM layer ids
m=lm.GPT(lm.LMConfig(attention="hash")).cuda()
seen=[]; real=lm.lsh_bucket_ids
lm.lsh_bucket_ids=lambda k,R: seen.append(real(k,R)) or seen[-1]
idx=torch.randint(0,50304,(4,8192),device="cuda")
with torch.no_grad(), torch.autocast("cuda",dtype=torch.bfloat16): m(idx)
for i,ids in enumerate(seen):
    c=torch.bincount(ids.flatten(),minlength=16).float()
    # per (b,h) collision fraction
    oh=torch.nn.functional.one_hot(ids,16).sum(1).float()  # (B,H,16)
    print("layer",i,"global hist",(c/c.sum()).cpu().numpy().round(3),"mean coll %.4f"%float((oh**2).sum(-1).mean()/T**2))

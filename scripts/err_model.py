"""Error model of the backward at D = 128 (tests/test_gpu_fullsize.py): fp64 gradients with
the kernel's two roundings applied one at a time — delta from the bf16 O, dS in bf16."""
import torch
torch.manual_seed(0)
T,D,nb=4096,128,64
def bf(x): return x.to(torch.bfloat16).double()
q,k,v,dO=(bf(torch.randn(T,D)) for _ in range(4))
ids=torch.randint(0,nb,(T,))
pos=torch.arange(T)
vis=(pos[:,None]>pos[None,:])&(ids[:,None]==ids[None,:])
sc=D**-0.5
s=(q@k.T)*sc
s=s.masked_fill(~vis,float('-inf'))
p=torch.softmax(s,-1).nan_to_num(0)
o=p@v
dp=dO@v.T
delta=(dO*o).sum(-1,keepdim=True)
ds=p*(dp-delta)
dk_ref=sc*ds.T@q
dq_ref=sc*ds@k
for name,dl,pr,dsr in [("exact",delta,p,ds),("O bf16 delta",(dO*bf(o)).sum(-1,keepdim=True),p,None),("dS bf16",delta,p,"bf"),("both",(dO*bf(o)).sum(-1,keepdim=True),p,"bf")]:
    d=pr*(dp-dl)
    if dsr=="bf": d=bf(d)
    dk=sc*d.T@q; dq=sc*d@k
    print(name,"dK err",float((dk-dk_ref).abs().max()),"dQ err",float((dq-dq_ref).abs().max()), "max|dK|",float(dk_ref.abs().max()))

import sys, time, torch, numpy as np
sys.path.insert(0,'.')
from paper_2510_01579_b200 import batched
from paper_2510_01579_b200.params import CacParams
P=45864; n=8
g=torch.Generator(device='cuda').manual_seed(0)
H=torch.complex(torch.randn(P,n,n,dtype=torch.float64,device='cuda',generator=g),torch.randn(P,n,n,dtype=torch.float64,device='cuda',generator=g))*0.5**0.5
lv=torch.tensor([-3,-1,1,3],dtype=torch.float64,device='cuda')/10**0.5
u=torch.complex(lv[torch.randint(0,4,(P,n),device='cuda',generator=g)], lv[torch.randint(0,4,(P,n),device='cuda',generator=g)])
seeds=torch.arange(P,device='cuda')
tau=2.0*(3/10**0.5+1/10**0.5)
for prec in ('fp32','fp64_exact'):
    r=batched.precode_vpp_batch(H,u,float(n),tau,seeds,CacParams(precision=prec)); torch.cuda.synchronize()
    t0=time.perf_counter()
    for _ in range(3): r=batched.precode_vpp_batch(H,u,float(n),tau,seeds,CacParams(precision=prec))
    torch.cuda.synchronize(); dt=(time.perf_counter()-t0)/3
    print(prec, f"VPP 8x8 16-QAM slot: {dt*1e3:.2f} ms  {P/dt/1e6:.2f} M prec/s", flush=True)

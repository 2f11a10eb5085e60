import sys, torch
sys.path.insert(0,'.')
from tools.parity_scale import batch
from paper_2510_01579_b200 import batched, _lib
from paper_2510_01579_b200.params import CacParams
P=45864
H,y,nv,seeds,_=batch(16,16,20.0,P,3)
for f in (1,2,4,8,128):
    prm=CacParams(f_mvm=f)
    batched.detect_cim_batch(H,y,nv,16,seeds,prm); torch.cuda.synchronize()
    _lib.profile_begin()
    for _ in range(3): batched.detect_cim_batch(H,y,nv,16,seeds,prm)
    pr=_lib.profile_end()
    print(f"f_mvm={f}: anneal {pr['anneal'][0]/3:.3f} ms", flush=True)

"""Quick device-resident throughput probe of detect_cim_batch (dev tool)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2510_01579_b200 import batched
from paper_2510_01579_b200.params import CacParams

def run(n_t, order, P, prec, reps=3):
    g = torch.Generator(device="cuda").manual_seed(0)
    H = (torch.randn(P, n_t, n_t, dtype=torch.float64, device="cuda", generator=g)
         + 1j * torch.randn(P, n_t, n_t, dtype=torch.float64, device="cuda", generator=g)) * 0.5 ** 0.5
    x = (torch.randint(0, 2, (P, n_t), device="cuda", generator=g) * 2 - 1).to(torch.complex128) / 2 ** 0.5
    s2 = n_t / 10 ** 2.0
    y = torch.einsum("prt,pt->pr", H, x) + (torch.randn(P, n_t, dtype=torch.complex128, device="cuda", generator=g)) * s2 ** 0.5
    nv = torch.full((P,), s2, dtype=torch.float64, device="cuda")
    seeds = torch.arange(P, dtype=torch.int64, device="cuda").to(torch.uint64)
    prm = CacParams(precision=prec)
    batched.detect_cim_batch(H, y, nv, order, seeds, prm)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); batched.detect_cim_batch(H, y, nv, order, seeds, prm); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    print(f"n_t={n_t} M={order} P={P} {prec}: {ms:.3f} ms  {P / ms * 1e3 / 1e6:.3f} Mdet/s", flush=True)

if len(sys.argv) > 1:
    run(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5]) if len(sys.argv) > 5 else 3)
else:
    for prec in ("fp32", "tf32", "fp64_exact"):
        run(16, 16, 45864 if prec != "fp64_exact" else 4096, prec)
        run(8, 16, 45864 if prec != "fp64_exact" else 4096, prec)

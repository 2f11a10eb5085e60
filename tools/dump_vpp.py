"""Dump precode_vpp_batch outputs for a fixed synthetic slot (dev tool):
python tools/dump_vpp.py out.npz"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2510_01579_b200 import batched  # noqa: E402
from paper_2510_01579_b200.params import CacParams  # noqa: E402
out = {}
for n, P in ((8, 8192), (4, 4096), (6, 4096)):
    g = torch.Generator(device='cuda').manual_seed(n)
    H = torch.complex(torch.randn(P, n, n, dtype=torch.float64, device='cuda', generator=g),
                      torch.randn(P, n, n, dtype=torch.float64, device='cuda', generator=g)) * 0.5 ** 0.5
    lv = torch.tensor([-3, -1, 1, 3], dtype=torch.float64, device='cuda') / 10 ** 0.5
    u = torch.complex(lv[torch.randint(0, 4, (P, n), device='cuda', generator=g)],
                      lv[torch.randint(0, 4, (P, n), device='cuda', generator=g)])
    seeds = torch.arange(P, device='cuda')
    tau = 2.0 * (3 / 10 ** 0.5 + 1 / 10 ** 0.5)
    for prec in ("fp32", "fp64_exact"):
        r = batched.precode_vpp_batch(H, u, float(n), tau, seeds, CacParams(precision=prec))
        for f in ("x", "v", "unnormalized_power"):
            out[f"{n}_{prec}_{f}"] = getattr(r, f).cpu().numpy()
np.savez(sys.argv[1], **out)

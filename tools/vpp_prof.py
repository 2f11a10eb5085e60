"""VPP slot time per kernel kind (dev tool)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2510_01579_b200 import batched, _lib  # noqa: E402
from paper_2510_01579_b200.params import CacParams  # noqa: E402
P = 45864; n = 8
g = torch.Generator(device='cuda').manual_seed(0)
H = torch.complex(torch.randn(P, n, n, dtype=torch.float64, device='cuda', generator=g),
                  torch.randn(P, n, n, dtype=torch.float64, device='cuda', generator=g)) * 0.5 ** 0.5
lv = torch.tensor([-3, -1, 1, 3], dtype=torch.float64, device='cuda') / 10 ** 0.5
u = torch.complex(lv[torch.randint(0, 4, (P, n), device='cuda', generator=g)],
                  lv[torch.randint(0, 4, (P, n), device='cuda', generator=g)])
seeds = torch.arange(P, device='cuda')
tau = 2.0 * (3 / 10 ** 0.5 + 1 / 10 ** 0.5)
prm = CacParams()
batched.precode_vpp_batch(H, u, float(n), tau, seeds, prm); torch.cuda.synchronize()
_lib.profile_begin()
for _ in range(3):
    batched.precode_vpp_batch(H, u, float(n), tau, seeds, prm)
pr = _lib.profile_end()
print(" ".join(f"{k}={v[0] / 3:.3f}ms/{v[1] // 3}" for k, v in pr.items() if v[1]))

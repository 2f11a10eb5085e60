"""VPP parity at scale (dev tool): fp32 / tf32 against the FP64-exact kernel
(bit-identical to the reference) on fresh synthetic 8x8 16-QAM problems --
identical perturbation vectors, and unnormalised power <= exact."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2510_01579_b200 import batched  # noqa: E402
from paper_2510_01579_b200.params import CacParams  # noqa: E402
for n, P in ((8, 45864), (4, 16384)):
    g = torch.Generator(device='cuda').manual_seed(100 + n)
    H = torch.complex(torch.randn(P, n, n, dtype=torch.float64, device='cuda', generator=g),
                      torch.randn(P, n, n, dtype=torch.float64, device='cuda', generator=g)) * 0.5 ** 0.5
    lv = torch.tensor([-3, -1, 1, 3], dtype=torch.float64, device='cuda') / 10 ** 0.5
    u = torch.complex(lv[torch.randint(0, 4, (P, n), device='cuda', generator=g)],
                      lv[torch.randint(0, 4, (P, n), device='cuda', generator=g)])
    seeds = torch.arange(P, device='cuda') * 7 + n
    tau = 2.0 * (3 / 10 ** 0.5 + 1 / 10 ** 0.5)
    res = {p: batched.precode_vpp_batch(H, u, float(n), tau, seeds, CacParams(precision=p))
           for p in ("fp64_exact", "fp32", "tf32")}
    ex = res["fp64_exact"]
    line = [f"VPP {n}x{n} 16-QAM P={P}:"]
    for p in ("fp32", "tf32"):
        r = res[p]
        same = (r.v == ex.v).all(-1).float().mean().item()
        le = (r.unnormalized_power <= ex.unnormalized_power * (1 + 1e-12)).float().mean().item()
        line.append(f"{p}: v identical {same:.4f}, power<=exact {le:.4f}")
    print("  ".join(line), flush=True)

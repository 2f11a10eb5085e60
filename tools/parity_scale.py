"""Throughput-mode parity at scale (dev tool): fp32 / tf32 anneals against the
FP64-exact kernel (bit-identical to the reference) on fresh synthetic REs.

    python tools/parity_scale.py [P]

Per config: fraction of REs whose final energy is <= the exact run's, the
fraction of identical decisions, and the SER of each mode."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_01579_b200 import batched  # noqa: E402
from paper_2510_01579_b200.params import CacParams  # noqa: E402


def batch(n_t, order, snr_db, P, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    H = torch.complex(torch.randn(P, n_t, n_t, dtype=torch.float64, device="cuda", generator=g),
                      torch.randn(P, n_t, n_t, dtype=torch.float64, device="cuda", generator=g)) * 0.5 ** 0.5
    m = int(round(order ** 0.5))
    lv = torch.arange(-(m - 1), m, 2, dtype=torch.float64, device="cuda") / (2 * (m * m - 1) / 3) ** 0.5
    ir = torch.randint(0, m, (P, n_t), device="cuda", generator=g)
    ii = torch.randint(0, m, (P, n_t), device="cuda", generator=g)
    x = torch.complex(lv[ir], lv[ii])
    s2 = n_t / 10 ** (snr_db / 10)
    nz = torch.complex(torch.randn(P, n_t, dtype=torch.float64, device="cuda", generator=g),
                       torch.randn(P, n_t, dtype=torch.float64, device="cuda", generator=g))
    y = torch.einsum("prt,pt->pr", H, x) + nz * (s2 / 2) ** 0.5
    nv = torch.full((P,), s2, dtype=torch.float64, device="cuda")
    seeds = torch.randint(0, 2**62, (P,), device="cuda", generator=g)
    truth = torch.stack([ir, ii], -1).to(torch.uint8)
    return H, y, nv, seeds, truth


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    for (n_t, order, snr) in ((8, 16, 20.0), (16, 16, 20.0), (16, 64, 25.0), (8, 4, 10.0)):
        H, y, nv, seeds, truth = batch(n_t, order, snr, P, 1234 + n_t + order)
        res = {p: batched.detect_cim_batch(H, y, nv, order, seeds, CacParams(precision=p))
               for p in ("fp64_exact", "fp32", "tf32")}
        ex = res["fp64_exact"]
        line = [f"{n_t}x{n_t} {order}-QAM {snr:.0f} dB P={P}:"]
        for p in ("fp64_exact", "fp32", "tf32"):
            r = res[p]
            ser = (r.x_idx != truth).any(-1).float().mean().item()
            le = (r.energy <= ex.energy * (1 + 1e-12)).float().mean().item()
            same = (r.x_idx == ex.x_idx).all(-1).all(-1).float().mean().item()
            line.append(f"{p}: E<=exact {le:.4f} same {same:.4f} SER {ser:.4f}")
        print("  ".join(line), flush=True)


if __name__ == "__main__":
    main()

"""Randomised shapes / parameters / modes through the batched detector, each
against the FP64-exact mode (dev tool): no launch errors, energy <= exact on
most REs, PACK == padded, fused paths consistent.

    python tools/fuzz_modes.py [n_cases]
"""
import os
import random
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2510_01579_b200 import batched  # noqa: E402
from paper_2510_01579_b200.params import CacParams  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    rnd = random.Random(int(os.environ.get("FUZZ_SEED", "7")))
    dev = torch.device("cuda", 0)
    bad = 0
    for case in range(n):
        n_t = rnd.choice([1, 2, 3, 4, 5, 6, 8, 9, 11, 12, 13, 16, 17, 20, 24, 28, 32])
        n_r = n_t + rnd.choice([0, 0, 1, 4])
        order = rnd.choice([4, 16, 64])
        snr = rnd.choice([5.0, 15.0, 25.0])
        na = rnd.choice([1, 3, 8, 12, 16, 20, 32, 40])
        kw = dict(n_anneals=na, f_mvm=rnd.choice([1, 2, 3]), n_steps=rnd.choice([64, 128, 200]))
        prec = rnd.choice(["fp32", "mixed", "tf32"])
        rng = rnd.choice(["numpy", "philox"])
        P = rnd.choice([1, 7, 300, 1001])
        H, y, nv, seeds, truth, _ = bench._synthetic_uplink(dev, P, n_t, order, snr, 1000 + case)
        if n_r != n_t:  # taller channel
            g = torch.Generator(device=dev).manual_seed(case)
            H = torch.complex(torch.randn(P, n_r, n_t, dtype=torch.float64, device=dev, generator=g),
                              torch.randn(P, n_r, n_t, dtype=torch.float64, device=dev, generator=g)) * 0.5 ** 0.5
            y = torch.complex(torch.randn(P, n_r, dtype=torch.float64, device=dev, generator=g),
                              torch.randn(P, n_r, dtype=torch.float64, device=dev, generator=g))
        try:
            ex = batched.detect_cim_batch(H, y, nv, order, seeds, CacParams(precision="fp64_exact", rng=rng, **kw))
            fa = batched.detect_cim_batch(H, y, nv, order, seeds, CacParams(precision=prec, rng=rng, **kw))
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            print(f"case {case} ERROR n_t={n_t} n_r={n_r} M={order} {kw} {prec} {rng} P={P}: {e}")
            bad += 1
            continue
        le = (fa.energy <= ex.energy * (1 + 1e-12)).float().mean().item()
        same = (fa.x_idx == ex.x_idx).all(-1).all(-1).float().mean().item()
        flag = "" if le >= (0.95 if prec != "tf32" else 0.9) else "  <-- LOW"
        bad += bool(flag)
        print(f"case {case}: n_t={n_t} n_r={n_r} M={order} {snr:.0f}dB {kw} {prec} {rng} P={P}: "
              f"E<=exact {le:.4f} same {same:.4f}{flag}", flush=True)
    print(f"{bad} suspicious of {n}")


if __name__ == "__main__":
    main()

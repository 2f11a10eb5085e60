"""Quick device-resident throughput probe of detect_cim_batch (dev tool).

    python tools/quick_bench.py [n_t order P precision reps n_anneals rng]

Prints the slot time and the per-kernel-kind times from the library's
CUDA-event hooks.  ISINGLINK_B200_LIB selects a variant build.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_01579_b200 import _lib, batched  # noqa: E402
from paper_2510_01579_b200.params import CacParams  # noqa: E402


def run(n_t, order, P, prec, reps=3, tag="", n_anneals=32, rng="numpy"):
    g = torch.Generator(device="cuda").manual_seed(0)
    H = (torch.randn(P, n_t, n_t, dtype=torch.float64, device="cuda", generator=g)
         + 1j * torch.randn(P, n_t, n_t, dtype=torch.float64, device="cuda", generator=g)) * 0.5 ** 0.5
    m = int(round(order ** 0.5))
    lv = (torch.arange(-(m - 1), m, 2, dtype=torch.float64, device="cuda")
          / (2 * (m * m - 1) / 3) ** 0.5)
    x = torch.complex(lv[torch.randint(0, m, (P, n_t), device="cuda", generator=g)],
                      lv[torch.randint(0, m, (P, n_t), device="cuda", generator=g)])
    s2 = n_t / 10 ** 2.0
    y = torch.einsum("prt,pt->pr", H, x) + (torch.randn(P, n_t, dtype=torch.complex128, device="cuda",
                                                        generator=g)) * s2 ** 0.5
    nv = torch.full((P,), s2, dtype=torch.float64, device="cuda")
    seeds = torch.arange(P, dtype=torch.int64, device="cuda").to(torch.uint64)
    prm = CacParams(precision=prec, n_anneals=n_anneals, rng=rng)
    r = batched.detect_cim_batch(H, y, nv, order, seeds, prm)
    torch.cuda.synchronize()
    ts = []
    _lib.profile_begin()
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        batched.detect_cim_batch(H, y, nv, order, seeds, prm)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    prof = _lib.profile_end()
    ms = min(ts)
    kk = " ".join(f"{k}={v[0] / reps:.3f}" for k, v in prof.items() if v[1])
    src = r.source.float().mean().item()
    print(f"{tag} n_t={n_t} M={order} P={P} N_a={n_anneals} {prec} {rng}: {ms:.3f} ms  {P / ms * 1e3 / 1e6:.3f} Mdet/s"
          f"  [{kk}] src_mean={src:.4f}", flush=True)


if __name__ == "__main__":
    tag = os.path.basename(os.path.dirname(os.environ.get("ISINGLINK_B200_LIB", "default/x")))
    if len(sys.argv) > 4:
        run(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4],
            int(sys.argv[5]) if len(sys.argv) > 5 else 3, tag,
            int(sys.argv[6]) if len(sys.argv) > 6 else 32,
            sys.argv[7] if len(sys.argv) > 7 else "numpy")
    else:
        for prec in ("fp32", "tf32", "fp64_exact"):
            run(16, 16, 45864 if prec != "fp64_exact" else 4096, prec, tag=tag)
            run(8, 16, 45864 if prec != "fp64_exact" else 4096, prec, tag=tag)

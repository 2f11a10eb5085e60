"""Anneal cost split (dev tool): k_anneal_fast time vs n_steps and f_mvm on a
full 16x16 16-QAM slot, separating the fixed prologue/epilogue cost from the
per-step Euler cost and the per-refresh tensor-core cost."""
import sys

import torch

sys.path.insert(0, '.')
from tools.parity_scale import batch  # noqa: E402
from paper_2510_01579_b200 import batched, _lib  # noqa: E402
from paper_2510_01579_b200.params import CacParams  # noqa: E402

P = 45864
H, y, nv, seeds, _ = batch(16, 16, 20.0, P, 3)
import os
PREC = os.environ.get("PREC", "fp32")
RNG = os.environ.get("RNG", "numpy")
for steps, f in ((2, 2), (32, 2), (128, 2), (256, 2), (128, 1), (128, 4), (128, 128), (256, 256), (4, 2), (8, 2)):
    prm = CacParams(f_mvm=f, n_steps=steps, precision=PREC, rng=RNG)
    batched.detect_cim_batch(H, y, nv, 16, seeds, prm)
    torch.cuda.synchronize()
    _lib.profile_begin()
    for _ in range(3):
        batched.detect_cim_batch(H, y, nv, 16, seeds, prm)
    pr = _lib.profile_end()
    print(f"{PREC} {RNG} n_steps={steps} f_mvm={f}: anneal {pr['anneal'][0] / 3:.3f} ms", flush=True)

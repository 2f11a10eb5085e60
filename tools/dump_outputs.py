"""Dump detect_cim_batch outputs (fp32) for a fixed synthetic slot, to compare
library variants bit-for-bit (dev tool):  python tools/dump_outputs.py out.npz"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_01579_b200 import batched  # noqa: E402
from paper_2510_01579_b200.params import CacParams  # noqa: E402
from tools.parity_scale import batch  # noqa: E402

out = {}
for (n_t, order, snr) in ((16, 16, 20.0), (8, 16, 15.0), (16, 64, 30.0)):
    H, y, nv, seeds, _ = batch(n_t, order, snr, 16384, 99 + n_t)
    r = batched.detect_cim_batch(H, y, nv, order, seeds, CacParams(precision="fp32"))
    key = f"{n_t}_{order}"
    for f in ("x_idx", "energy", "source", "anneal_index", "diverged"):
        out[f"{key}_{f}"] = getattr(r, f).cpu().numpy()
np.savez(sys.argv[1], **out)
if len(sys.argv) > 2:
    ref = np.load(sys.argv[2])
    bad = [k for k in out if not np.array_equal(out[k], ref[k])]
    print("identical to", sys.argv[2] if not bad else f"DIFFERS in {bad}")

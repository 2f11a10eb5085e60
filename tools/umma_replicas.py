"""tcgen05 vs mma.sync anneal at larger replica counts (dev tool): one
problem per CTA when n_anneals = 64 (M = 64 rows, no wasted MACs)."""
import os
import sys

import torch

sys.path.insert(0, '.')
from tools.parity_scale import batch  # noqa: E402
from paper_2510_01579_b200 import batched, _lib  # noqa: E402
from paper_2510_01579_b200.params import CacParams  # noqa: E402

tag = "umma" if os.environ.get("ISINGLINK_UMMA") == "1" else "mma.sync"
P = 45864
for n_t, order, snr in ((16, 16, 20.0), (16, 64, 30.0)):
    H, y, nv, seeds, _ = batch(n_t, order, snr, P, 3)
    for na in (32, 64, 128):
        prm = CacParams(n_anneals=na)
        r = batched.detect_cim_batch(H, y, nv, order, seeds, prm)
        torch.cuda.synchronize()
        _lib.profile_begin()
        for _ in range(3):
            r = batched.detect_cim_batch(H, y, nv, order, seeds, prm)
        pr = _lib.profile_end()
        print(f"{tag} n_t={n_t} M={order} N_a={na}: anneal {pr['anneal'][0] / 3:.3f} ms "
              f"src_mean={r.source.float().mean().item():.4f} e_mean={r.energy.mean().item():.6f}", flush=True)

"""e2e (host-buffer) throughput of il_detect_cim_host vs chunk count (dev tool)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_01579_b200 import batched  # noqa: E402
from paper_2510_01579_b200.params import CacParams  # noqa: E402
from tools.parity_scale import batch  # noqa: E402

P = 45864
H, y, nv, seeds, _ = batch(16, 16, 20.0, P, 7)
Hh, yh, nvh, sh = (t.cpu().pin_memory() for t in (H, y, nv, seeds))
out = None
prm = CacParams()
# raw H2D bandwidth of the slot's inputs
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    Hh.to("cuda", non_blocking=True)
torch.cuda.synchronize()
print(f"H2D pinned: {3 * Hh.numel() * 16 / (time.perf_counter() - t0) / 1e9:.1f} GB/s", flush=True)
for n in (1, 2, 4, 8, 12, 16, 24, 32):
    batched.detect_cim_host(Hh, yh, nvh, 16, sh, prm, n_chunks=n)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        batched.detect_cim_host(Hh, yh, nvh, 16, sh, prm, n_chunks=n)
        ts.append(time.perf_counter() - t0)
    print(f"n_chunks={n:3d}: {min(ts) * 1e3:.2f} ms  {P / min(ts) / 1e6:.2f} M det/s", flush=True)

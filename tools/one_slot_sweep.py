"""One-slot-at-a-time e2e vs chunk count (dev tool)."""
import sys
import time
import torch
sys.path.insert(0, '.')
from paper_2510_01579_b200 import batched  # noqa: E402
from paper_2510_01579_b200.params import CacParams  # noqa: E402
from tools.parity_scale import batch  # noqa: E402
P = 45864
H, y, nv, seeds, _ = batch(16, 16, 20.0, P, 7)
Hh, yh, nvh, sh = (t.cpu().pin_memory() for t in (H, y, nv, seeds))
prm = CacParams()
out = batched.detect_cim_host(Hh, yh, nvh, 16, sh, prm)
for c in (0, 2, 3, 4, 6, 8, 12, 16, 24):
    batched.detect_cim_host(Hh, yh, nvh, 16, sh, prm, n_chunks=c, out=out)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        t0 = time.perf_counter()
        batched.detect_cim_host(Hh, yh, nvh, 16, sh, prm, n_chunks=c, out=out)
        best = min(best, time.perf_counter() - t0)
    print(f"n_chunks={c}: {best * 1e3:.3f} ms", flush=True)

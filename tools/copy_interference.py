"""Do concurrent H2D copies slow the device-resident detection? (dev tool)"""
import sys
import time

import torch

sys.path.insert(0, '.')
from tools.parity_scale import batch  # noqa: E402
from paper_2510_01579_b200 import batched, _lib  # noqa: E402
from paper_2510_01579_b200.params import CacParams  # noqa: E402

P = 45864
H, y, nv, seeds, _ = batch(16, 16, 20.0, P, 7)
prm = CacParams()
host = torch.empty(200 * 2 ** 20, dtype=torch.uint8).pin_memory()
dev = torch.empty_like(host, device="cuda")
side = torch.cuda.Stream()
batched.detect_cim_batch(H, y, nv, 16, seeds, prm)
torch.cuda.synchronize()
for copy in (False, True, False, True):
    _lib.profile_begin()
    t0 = time.perf_counter()
    if copy:
        with torch.cuda.stream(side):
            dev.copy_(host, non_blocking=True)
    batched.detect_cim_batch(H, y, nv, 16, seeds, prm)
    torch.cuda.synchronize()
    pr = _lib.profile_end()
    print(f"copy={copy}: wall {1e3 * (time.perf_counter() - t0):.3f} ms  "
          + " ".join(f"{k}={v[0]:.3f}" for k, v in pr.items() if v[1]), flush=True)

"""Per-call timing of streamed slots (dev tool)."""
import os
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
outs = [batched.detect_cim_host(Hh, yh, nvh, 16, sh, prm) for _ in range(2)]
torch.cuda.synchronize()
for rep in range(3):
    K = 8
    t0 = time.perf_counter()
    prev = None
    log = []
    for k in range(K):
        a = time.perf_counter()
        tk = batched.detect_cim_host_submit(Hh, yh, nvh, 16, sh, prm, out=outs[k % 2])
        b = time.perf_counter()
        if prev is not None:
            prev.wait()
        c = time.perf_counter()
        log.append(f"{(b - a) * 1e3:.2f}/{(c - b) * 1e3:.2f}")
        prev = tk
    prev.wait()
    ms = (time.perf_counter() - t0) * 1e3 / K
    print(f"rep {rep}: {ms:.3f} ms/slot  submit/wait ms: {' '.join(log)}", flush=True)

"""Streamed slots: first slot auto-chunked, later slots with n_chunks = c (dev tool)."""
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
for c in (0, 1, 2, 4, 8):
    for rep in range(2):
        K = 10
        t0 = time.perf_counter()
        prev = None
        for k in range(K):
            tk = batched.detect_cim_host_submit(Hh, yh, nvh, 16, sh, prm, out=outs[k % 2],
                                                n_chunks=(0 if k == 0 else c))
            if prev is not None:
                prev.wait()
            prev = tk
        prev.wait()
        print(f"later slots n_chunks={c}: {(time.perf_counter() - t0) * 1e3 / K:.3f} ms/slot", flush=True)

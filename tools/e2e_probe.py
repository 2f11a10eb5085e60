"""Where does the e2e (host-buffer) time go? (dev tool)"""
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
prm = CacParams()


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


print(f"H2D of all inputs: {t(lambda: [x.to('cuda', non_blocking=True) for x in (Hh, yh, nvh, sh)]):.2f} ms")
print(f"device-resident detect: {t(lambda: batched.detect_cim_batch(H, y, nv, 16, seeds, prm)):.2f} ms")
for n in (1, 0, 12, 16):
    print(f"host pipeline n_chunks={n}: {t(lambda: batched.detect_cim_host(Hh, yh, nvh, 16, sh, prm, n_chunks=n)):.2f} ms")
# chunked device-resident (no copies) on two streams: chunking overhead alone
ch = (P + 11) // 12
s = [torch.cuda.Stream(), torch.cuda.Stream()]


def chunked():
    for c in range(12):
        with torch.cuda.stream(s[c & 1]):
            sl = slice(c * ch, min(P, (c + 1) * ch))
            batched.detect_cim_batch(H[sl], y[sl], nv[sl], 16, seeds[sl], prm)


print(f"device-resident, 12 chunks on 2 streams: {t(chunked):.2f} ms")

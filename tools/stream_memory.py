"""Device memory over many streamed slots (dev tool): the pool must plateau."""
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
free0 = torch.cuda.mem_get_info()[0]
prev = None
t0 = time.perf_counter()
for k in range(200):
    n = P if k % 3 else P // 2 + k  # varying sizes
    tk = batched.detect_cim_host_submit(Hh[:n], yh[:n], nvh[:n], 16, sh[:n], prm)
    if prev is not None:
        prev.wait()
    prev = tk
    if k % 50 == 49:
        print(f"slot {k + 1}: device free {torch.cuda.mem_get_info()[0] / 2**30:.2f} GiB "
              f"(start {free0 / 2**30:.2f}), {(time.perf_counter() - t0) * 1e3 / (k + 1):.2f} ms/slot", flush=True)
prev.wait()

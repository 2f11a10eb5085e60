"""Host enqueue time vs device time per detect_cim_batch call at small P
(the per-rank share of a slot at N GPUs) -- dev tool.

    python tools/host_overhead.py [P ...]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2510_01579_b200 import batched  # noqa: E402
from paper_2510_01579_b200.params import CacParams  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    prm = CacParams()
    for P in [int(a) for a in sys.argv[1:]] or [5733, 11466, 45864]:
        H, y, nv, seeds, _ = bench.headline_slot(dev, 0, P)
        for _ in range(3):
            r = batched.detect_cim_batch(H, y, nv, 16, seeds, prm)
            batched.gray_demap(r.x_idx, 2)
        torch.cuda.synchronize()
        n = 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(n):
            r = batched.detect_cim_batch(H, y, nv, 16, seeds, prm)
            batched.gray_demap(r.x_idx, 2)
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"P={P}: host enqueue {1e3 * (t1 - t0) / n:.3f} ms/step, device {e0.elapsed_time(e1) / n:.3f} ms/step, "
              f"wall {1e3 * (t2 - t0) / n:.3f} ms/step", flush=True)


if __name__ == "__main__":
    main()

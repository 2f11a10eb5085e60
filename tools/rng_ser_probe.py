"""SER with the numpy-stream and the Philox initial states on the same
channels, each with two independent seedings (dev tool): is a gap between
the generators larger than the gap between two seedings of one generator?

    python tools/rng_ser_probe.py [P]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2510_01579_b200 import batched  # noqa: E402
from paper_2510_01579_b200.params import CacParams  # noqa: E402


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
    dev = torch.device("cuda", 0)
    for n_t, order, snr, na in ((8, 16, 30.0, 32), (16, 16, 30.0, 32), (16, 64, 30.0, 32), (8, 16, 25.0, 8)):
        H, y, nv, seeds, truth, _ = bench._synthetic_uplink(dev, P, n_t, order, snr, 900 + n_t)
        line = [f"{n_t}x{n_t} {order}-QAM {snr:.0f} dB N_a={na} P={P}:"]
        for rng in ("numpy", "philox"):
            for k, sd in enumerate((seeds, seeds ^ 0x5DEECE66D)):
                r = batched.detect_cim_batch(H, y, nv, order, sd, CacParams(n_anneals=na, rng=rng))
                ser = (r.x_idx != truth).any(-1).float().mean().item()
                div = r.diverged.float().mean().item()
                src = r.source.float().mean().item()
                line.append(f"{rng}#{k} SER {ser:.5f} div {div:.3f} anneal-src {src:.4f}")
        print("  ".join(line), flush=True)


if __name__ == "__main__":
    main()

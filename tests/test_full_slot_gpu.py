"""GPU parity on FULL slots (273 PRB x 12 subcarriers x 14 symbols = 45,864
REs): the FP32 throughput mode -- the arithmetic the headline number is
measured in -- against the FP64-exact kernel, which is bit-identical to the
reference's compiled kernel (tests/test_gpu_parity.py pins it to the
reference fixtures).

Gate (north_star): the final energy is <= the exact run's on >= 99% of the
REs.  The fraction of identical decisions and both SERs are printed.
References: detect_cim (detector.py:57-82) over solve_batch
(solver.py:238-279); precode_vpp (precoder.py:93-146).
"""

import math
import os
import sys

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu

SLOT = 273 * 12 * 14
# energies are FP64 residuals ||y - H x||^2 recomputed for the decided x;
# an identical decision reproduces the exact run's energy bit for bit
ENERGY_RTOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _ready(built_lib):
    assert torch.cuda.is_available()


def _compare(tag, fa, ex, truth):
    e_fa, e_ex = fa.energy.cpu().numpy(), ex.energy.cpu().numpy()
    le = float(np.mean(e_fa <= e_ex * (1 + ENERGY_RTOL)))
    same = (fa.x_idx == ex.x_idx).all(-1).all(-1).float().mean().item()
    ser_fa = (fa.x_idx != truth).any(-1).float().mean().item()
    ser_ex = (ex.x_idx != truth).any(-1).float().mean().item()
    print(f"{tag}: P={len(e_fa)} energy<=exact {le:.5f} identical decisions {same:.5f} "
          f"SER fp32 {ser_fa:.5f} exact {ser_ex:.5f}")
    assert len(e_fa) == SLOT
    assert le >= 0.99, (tag, le)
    return le, same


def test_headline_slot_16x16_16qam_20db():
    """The bench's own workload (bench.headline_slot): the slot the credited
    detections/s figure is measured on."""
    import bench
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    H, y, nv, seeds, truth = bench.headline_slot(torch.device("cuda", torch.cuda.current_device()))
    ex = batched.detect_cim_batch(H, y, nv, 16, seeds, CacParams(precision="fp64_exact"))
    fa = batched.detect_cim_batch(H, y, nv, 16, seeds, CacParams(precision="fp32"))
    _, same = _compare("16x16 16-QAM 20 dB (headline)", fa, ex, truth)
    assert same >= 0.99


def test_headline_slot_mixed_mode():
    """The "mixed" precision mode (coupling product's third split pass
    dropped after 16 steps) on the headline slot: same >= 99% energy gate."""
    import bench
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    H, y, nv, seeds, truth = bench.headline_slot(torch.device("cuda", torch.cuda.current_device()))
    ex = batched.detect_cim_batch(H, y, nv, 16, seeds, CacParams(precision="fp64_exact"))
    fa = batched.detect_cim_batch(H, y, nv, 16, seeds, CacParams(precision="mixed"))
    _, same = _compare("16x16 16-QAM 20 dB (headline), mixed", fa, ex, truth)
    assert same >= 0.99


@pytest.mark.parametrize("n_t,order,snr", [(8, 16, 20.0), (16, 64, 25.0)])
def test_full_slot_uplink(n_t, order, snr):
    import bench
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    dev = torch.device("cuda", torch.cuda.current_device())
    H, y, nv, seeds, truth, _ = bench._synthetic_uplink(dev, SLOT, n_t, order, snr, 100 + n_t + order)
    ex = batched.detect_cim_batch(H, y, nv, order, seeds, CacParams(precision="fp64_exact"))
    fa = batched.detect_cim_batch(H, y, nv, order, seeds, CacParams(precision="fp32"))
    _, same = _compare(f"{n_t}x{n_t} {order}-QAM {snr:.0f} dB", fa, ex, truth)
    assert same >= 0.99


def test_full_slot_vpp_8x8_16qam():
    """Downlink: the perturbation search on a full slot of 8x8 problems; the
    fp32 transmit power is <= the exact run's on >= 99% of the problems."""
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    g = torch.Generator(device="cuda").manual_seed(4)
    P, n = SLOT, 8
    H = torch.complex(torch.randn(P, n, n, dtype=torch.float64, device="cuda", generator=g),
                      torch.randn(P, n, n, dtype=torch.float64, device="cuda", generator=g)) * math.sqrt(0.5)
    lv = torch.tensor([-3.0, -1.0, 1.0, 3.0], dtype=torch.float64, device="cuda") / math.sqrt(10.0)
    u = torch.complex(lv[torch.randint(0, 4, (P, n), device="cuda", generator=g)],
                      lv[torch.randint(0, 4, (P, n), device="cuda", generator=g)])
    tau = float(2.0 * (lv[-1] + (lv[1] - lv[0]) / 2))
    seeds = torch.arange(P, dtype=torch.int64, device="cuda")
    ex = batched.precode_vpp_batch(H, u, float(n), tau, seeds, CacParams(precision="fp64_exact"))
    fa = batched.precode_vpp_batch(H, u, float(n), tau, seeds, CacParams(precision="fp32"))
    p_ex = ex.unnormalized_power.cpu().numpy()
    p_fa = fa.unnormalized_power.cpu().numpy()
    le = float(np.mean(p_fa <= p_ex * (1 + 1e-11)))
    same = (fa.v == ex.v).all(-1).float().mean().item()
    gain = float(np.mean(p_ex) / np.mean(p_fa))
    print(f"8x8 16-QAM VPP: P={P} power<=exact {le:.5f} identical v {same:.5f} "
          f"mean power exact/fp32 {gain:.6f}")
    assert le >= 0.99
    assert same >= 0.99

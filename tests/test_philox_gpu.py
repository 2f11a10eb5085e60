"""Counter-based initial states (CacParams.rng = "philox", north_star's
"Philox counter-based RNG"): Philox4x32-10 keyed by the per-problem seeds
instead of the replayed numpy streams.  Not the reference's streams, so the
parity bars are (a) the north_star energy gate "under replayed Philox seeds":
the FP32 kernel against the FP64 reference dynamics (fp64_exact) started from
the SAME Philox states, and (b) statistical agreement of the symbol error
rate with the numpy-stream mode.  References: solver.py:182-187 (initial
states), solver.py:238-279 (solve_batch), detector.py:57-82 (detect_cim).
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


@pytest.fixture(scope="module", autouse=True)
def _ready(built_lib):
    assert torch.cuda.is_available()


def _ser(r, truth):
    return (r.x_idx != truth).any(-1).float().mean().item()


@pytest.mark.parametrize("n_t,order,snr,n_anneals", [(16, 16, 20.0, 32), (8, 16, 20.0, 32),
                                                     (16, 64, 30.0, 8), (6, 16, 15.0, 16)])
def test_philox_energy_gate_against_fp64(n_t, order, snr, n_anneals):
    import bench
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    dev = torch.device("cuda", torch.cuda.current_device())
    P = 16384
    H, y, nv, seeds, truth, _ = bench._synthetic_uplink(dev, P, n_t, order, snr, 300 + n_t)
    ex = batched.detect_cim_batch(H, y, nv, order, seeds,
                                  CacParams(n_anneals=n_anneals, precision="fp64_exact", rng="philox"))
    fa = batched.detect_cim_batch(H, y, nv, order, seeds,
                                  CacParams(n_anneals=n_anneals, precision="fp32", rng="philox"))
    le = (fa.energy <= ex.energy * (1 + 1e-12)).float().mean().item()
    same = (fa.x_idx == ex.x_idx).all(-1).all(-1).float().mean().item()
    print(f"philox {n_t}x{n_t} {order}-QAM N_a={n_anneals}: energy<=fp64 {le:.5f} identical {same:.5f} "
          f"SER fp32 {_ser(fa, truth):.5f} fp64 {_ser(ex, truth):.5f}")
    assert le >= 0.99
    assert same >= 0.99


def test_philox_ser_matches_numpy_streams():
    """Same channel draws, different initial-state generator: the SERs agree
    within the binomial noise of the difference (3 sigma)."""
    import bench
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    dev = torch.device("cuda", torch.cuda.current_device())
    H, y, nv, seeds, truth = bench.headline_slot(dev)
    a = batched.detect_cim_batch(H, y, nv, 16, seeds, CacParams(rng="numpy"))
    b = batched.detect_cim_batch(H, y, nv, 16, seeds, CacParams(rng="philox"))
    pa, pb = _ser(a, truth), _ser(b, truth)
    P = truth.shape[0]
    sigma = math.sqrt((pa * (1 - pa) + pb * (1 - pb)) / P)
    print(f"headline slot SER numpy {pa:.5f} philox {pb:.5f} (3 sigma {3 * sigma:.5f})")
    assert abs(pa - pb) <= 3 * sigma


def test_philox_packed_equals_padded():
    import bench
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    dev = torch.device("cuda", torch.cuda.current_device())
    H, y, nv, seeds, _, _ = bench._synthetic_uplink(dev, 1001, 16, 64, 30.0, 77)
    prm = CacParams(n_anneals=8, rng="philox")
    old = os.environ.get("ISINGLINK_PACK")
    try:
        os.environ["ISINGLINK_PACK"] = "1"
        a = batched.detect_cim_batch(H, y, nv, 64, seeds, prm)
        os.environ["ISINGLINK_PACK"] = "0"
        b = batched.detect_cim_batch(H, y, nv, 64, seeds, prm)
    finally:
        if old is None:
            os.environ.pop("ISINGLINK_PACK", None)
        else:
            os.environ["ISINGLINK_PACK"] = old
    for f in ("x_idx", "energy", "anneal_index", "diverged"):
        assert torch.equal(getattr(a, f), getattr(b, f)), f


def test_philox_vpp_runs_and_gates():
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    g = torch.Generator(device="cuda").manual_seed(21)
    P, n = 8192, 8
    H = torch.complex(torch.randn(P, n, n, dtype=torch.float64, device="cuda", generator=g),
                      torch.randn(P, n, n, dtype=torch.float64, device="cuda", generator=g)) * math.sqrt(0.5)
    lv = torch.tensor([-3.0, -1.0, 1.0, 3.0], dtype=torch.float64, device="cuda") / math.sqrt(10.0)
    u = torch.complex(lv[torch.randint(0, 4, (P, n), device="cuda", generator=g)],
                      lv[torch.randint(0, 4, (P, n), device="cuda", generator=g)])
    tau = float(2.0 * (lv[-1] + (lv[1] - lv[0]) / 2))
    seeds = torch.arange(P, dtype=torch.int64, device="cuda")
    ex = batched.precode_vpp_batch(H, u, float(n), tau, seeds, CacParams(precision="fp64_exact", rng="philox"))
    fa = batched.precode_vpp_batch(H, u, float(n), tau, seeds, CacParams(rng="philox"))
    le = float(np.mean(fa.unnormalized_power.cpu().numpy() <= ex.unnormalized_power.cpu().numpy() * (1 + 1e-11)))
    assert le >= 0.99


def test_rng_validation():
    from paper_2510_01579_b200.params import CacParams
    with pytest.raises(ValueError):
        CacParams(rng="mt19937").validate()

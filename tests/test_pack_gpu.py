"""Problems of n_anneals <= 8 run two per warp in the fast anneal kernel
(PACK: accumulator rows g are one problem's anneals, rows g + 8 the next
problem's).  Each anneal's trajectory depends only on its own seed stream
and its problem's couplings, and every tensor-core row sum is formed from
that row's operands alone, so the packed layout must reproduce the padded
16-row layout (ISINGLINK_PACK=0, the round-1 path) bit for bit: decisions,
energies, selected anneal, divergence counts, and the instrumented
steps / mvms counters.  References: solver.py:238-279 (solve_batch),
detector.py:57-82 (detect_cim), _kernel.pyx:85-97 (steps / mvms).
"""

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


def _both(fn):
    """fn() with the packed layout and with ISINGLINK_PACK=0."""
    old = os.environ.get("ISINGLINK_PACK")
    try:
        os.environ["ISINGLINK_PACK"] = "1"
        a = fn()
        torch.cuda.synchronize()
        os.environ["ISINGLINK_PACK"] = "0"
        b = fn()
        torch.cuda.synchronize()
    finally:
        if old is None:
            os.environ.pop("ISINGLINK_PACK", None)
        else:
            os.environ["ISINGLINK_PACK"] = old
    return a, b


# (n_t, order, snr, n_anneals, P): screened epilogue (N >= 24), FP64 epilogue
# (N = 16), inert padding spins (n_t = 6, 10), fewer than 8 anneals, odd P
# (the last warp holds a single problem)
CASES = [(16, 64, 30.0, 8, 2001), (8, 16, 20.0, 8, 1537), (6, 16, 15.0, 5, 999),
         (10, 4, 10.0, 8, 1024), (16, 16, 20.0, 3, 777), (1, 4, 10.0, 8, 257),
         (24, 16, 20.0, 8, 301), (32, 4, 15.0, 8, 129)]


@pytest.mark.parametrize("precision", ["fp32", "mixed", "tf32"])
@pytest.mark.parametrize("n_t,order,snr,n_anneals,P", CASES)
def test_detect_cim_packed_equals_padded(n_t, order, snr, n_anneals, P, precision):
    import bench
    from paper_2510_01579_b200 import _lib, batched
    from paper_2510_01579_b200.params import CacParams
    dev = torch.device("cuda", torch.cuda.current_device())
    H, y, nv, seeds, truth, _ = bench._synthetic_uplink(dev, P, n_t, order, snr, 7 + n_t + n_anneals)
    prm = CacParams(n_anneals=n_anneals, precision=precision)
    assert _lib.anneal_kernel(2 * n_t, prm) != "exact"
    a, b = _both(lambda: batched.detect_cim_batch(H, y, nv, order, seeds, prm))
    for f in ("x_idx", "energy", "source", "anneal_index", "diverged"):
        assert torch.equal(getattr(a, f), getattr(b, f)), f
    ser = (a.x_idx != truth).any(-1).float().mean().item()
    print(f"{n_t}x{n_t} {order}-QAM N_a={n_anneals} P={P} {precision}: packed == padded, SER {ser:.4f}")


@pytest.mark.parametrize("n_t,n_anneals", [(16, 8), (8, 6), (7, 8)])
def test_solve_batch_counts_packed_equals_padded(n_t, n_anneals):
    """Instrumented solve_batch (every anneal's FP64 energy, steps and mvms)."""
    import bench
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    dev = torch.device("cuda", torch.cuda.current_device())
    P = 513
    H, y, nv, seeds, _, _ = bench._synthetic_uplink(dev, P, n_t, 16, 12.0, 40 + n_t)
    x_idx, energy, _ = batched.mmse_batch(H, y, nv, 16)
    ising = batched.build_ising_batch(H, y, x_idx, 16)
    prm = CacParams(n_anneals=n_anneals, precision="fp32")
    a, b = _both(lambda: batched.solve_batch(ising["G"], ising["g_diag"], ising["b"], ising["offset"],
                                             energy, ising["eps_scale"], seeds, prm, counts=True))
    for f in ("best_spins", "best_energy", "best_index", "diverged", "steps", "mvms"):
        assert torch.equal(getattr(a, f), getattr(b, f)), f
    assert a.steps.shape == (P, n_anneals)


def test_packed_vpp_equals_padded():
    """Downlink perturbation search with 8 anneals per stage."""
    import math
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    g = torch.Generator(device="cuda").manual_seed(9)
    P, n = 1501, 8
    H = torch.complex(torch.randn(P, n, n, dtype=torch.float64, device="cuda", generator=g),
                      torch.randn(P, n, n, dtype=torch.float64, device="cuda", generator=g)) * math.sqrt(0.5)
    lv = torch.tensor([-3.0, -1.0, 1.0, 3.0], dtype=torch.float64, device="cuda") / math.sqrt(10.0)
    u = torch.complex(lv[torch.randint(0, 4, (P, n), device="cuda", generator=g)],
                      lv[torch.randint(0, 4, (P, n), device="cuda", generator=g)])
    tau = float(2.0 * (lv[-1] + (lv[1] - lv[0]) / 2))
    seeds = torch.arange(P, dtype=torch.int64, device="cuda")
    for stages, rng in ((1, "numpy"), (2, "numpy"), (2, "philox")):
        prm = CacParams(n_anneals=8, precision="fp32", rng=rng)
        a, b = _both(lambda: batched.precode_vpp_batch(H, u, float(n), tau, seeds, prm, n_stages=stages))
        assert torch.equal(a.v, b.v), (stages, rng)
        assert np.array_equal(a.unnormalized_power.cpu().numpy(), b.unnormalized_power.cpu().numpy())
        assert torch.equal(a.diverged, b.diverged)

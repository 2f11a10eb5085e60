"""GPU: MMGaP-E (detect_cim_multi, detector.py:85-134) and the batched
MMSE-SIC (linear.py:78-106) against the reference fixtures
(tests/golden/m*.npz, made by the real reference) and the oracle."""

import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import isinglink_oracle as orc

pytestmark = pytest.mark.gpu

MULTI_SETS = ["m8x8_16qam_15db", "m16x16_16qam_20db"]


@pytest.fixture(scope="module", autouse=True)
def _lib_ready(built_lib):
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return built_lib


@pytest.mark.parametrize("name", MULTI_SETS)
def test_mmse_sic_bit_exact_decisions(name):
    from paper_2510_01579_b200 import batched
    d = load_golden(f"{name}.npz")
    x, e, st = batched.mmse_sic_batch(d["H"], d["y"], d["noise_var"], int(d["order"]))
    assert np.all(st.cpu().numpy() == 0)
    assert np.array_equal(x.cpu().numpy(), d["x_sic"])
    np.testing.assert_allclose(e.cpu().numpy(), d["e_sic"], rtol=1e-12)


def test_mmse_sic_random_shapes_match_oracle():
    from paper_2510_01579_b200 import batched
    for (nr, nt, order, snr) in ((4, 4, 16, 12.0), (12, 8, 64, 22.0), (6, 3, 4, 6.0),
                                 (24, 20, 16, 20.0)):
        levels, _ = orc.qam(order)
        Hs, ys, ss, want = [], [], [], []
        for t in range(16):
            H, y, s2, _ = orc.uplink_instance(9, snr, 0, t, nr, nt, order)
            x, _ = orc.mmse_sic(H, y, s2, levels)
            Hs.append(H); ys.append(y); ss.append(s2)
            want.append(np.stack([orc.level_index(x.real, levels), orc.level_index(x.imag, levels)], -1))
        x, _, _ = batched.mmse_sic_batch(np.array(Hs), np.array(ys), np.array(ss), order)
        assert np.array_equal(x.cpu().numpy(), np.array(want)), (nr, nt)


@pytest.mark.parametrize("name", MULTI_SETS)
def test_detect_cim_multi_exact_matches_reference(name):
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    d = load_golden(f"{name}.npz")
    r = batched.detect_cim_multi_batch(d["H"], d["y"], d["noise_var"], int(d["order"]), d["seed"],
                                       CacParams(precision="fp64_exact"), int(d["n_stages"]))
    assert np.array_equal(r.x_idx.cpu().numpy(), d["x_hat"])
    np.testing.assert_allclose(r.energy.cpu().numpy(), d["energy"], rtol=1e-12)
    assert np.array_equal(r.source.cpu().numpy(), d["source"])
    assert np.array_equal(r.anneal_index.cpu().numpy(), d["anneal_index"])
    assert np.array_equal(r.diverged.cpu().numpy(), d["diverged"])


@pytest.mark.parametrize("name", MULTI_SETS)
def test_detect_cim_multi_fast_energy_parity(name):
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    d = load_golden(f"{name}.npz")
    r = batched.detect_cim_multi_batch(d["H"], d["y"], d["noise_var"], int(d["order"]), d["seed"],
                                       CacParams(precision="fp32"), int(d["n_stages"]))
    e = r.energy.cpu().numpy()
    assert (e <= d["energy"] * (1 + 1e-12)).mean() >= 0.99
    # never worse than either baseline
    assert np.all(e <= d["e_sic"] * (1 + 1e-12))


def test_multi_single_mmse_chain_is_detect_cim():
    """detector.py:96-99: chains=("mmse",), one stage reproduces detect_cim."""
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    d = load_golden("d8x8_16qam_20db.npz")
    for prec in ("fp64_exact", "fp32"):
        prm = CacParams(precision=prec)
        a = batched.detect_cim_batch(d["H"], d["y"], d["noise_var"], int(d["order"]), d["seed"], prm)
        b = batched.detect_cim_multi_batch(d["H"], d["y"], d["noise_var"], int(d["order"]),
                                           d["seed"], prm, 1, chains=("mmse",))
        for f in ("x_idx", "energy", "source", "anneal_index", "diverged"):
            assert torch.equal(getattr(a, f), getattr(b, f)), (prec, f)


def test_api_detect_cim_multi_hooks_and_fused_agree():
    from paper_2510_01579_b200 import api
    from paper_2510_01579_b200.params import CacParams
    d = load_golden("m8x8_16qam_15db.npz")
    c = api.make_qam(int(d["order"]))
    for i in range(6):
        inst = api.MimoInstance(H=d["H"][i], y=d["y"][i], constellation=c,
                                noise_var=float(d["noise_var"][i]))
        prm = CacParams(precision="fp64_exact")
        log = []
        a = api.detect_cim_multi(inst, prm, n_stages=2, seed=int(d["seed"][i]))
        b = api.detect_cim_multi(inst, prm, n_stages=2, seed=int(d["seed"][i]), stage_log=log)
        assert np.array_equal(a.x_hard, b.x_hard) and a.energy == b.energy
        assert a.source == b.source and a.anneal_index == b.anneal_index
        assert len(log) == 4 and [s for _, s, _ in log] == [0, 1, 0, 1]
        sic = api.detect_mmse_sic(inst)
        assert sic.source == "mmse_sic" and a.energy <= sic.energy

"""CPU: pin the oracle to the real reference before trusting it.

The golden fixtures (tests/golden/*.npz) were produced by the reference
package itself with its compiled Cython kernel (tests/golden/make_golden.py).
The oracle must reproduce them: run_anneals bit-for-bit, detections exactly,
Ising coefficients to rounding.  When the compiled reference kernel is
present in oracle/_ref (built here by `make -C oracle ref`), the C oracle
is also checked against it on fresh random problems.
"""

import numpy as np
import pytest

from conftest import load_golden
from oracle import isinglink_oracle as orc

DET_SETS = ["d8x8_qpsk_10db", "d8x8_16qam_20db", "d16x16_16qam_20db", "d16x16_64qam_25db"]


def _anneal_case(k):
    z = load_golden("anneals.npz")
    g = lambda n: z[f"c{k}_{n}"]
    return g


@pytest.mark.parametrize("k", range(11))
def test_c_oracle_run_anneals_bit_exact(k):
    g = _anneal_case(k)
    pr = g("prm")
    out = orc.run_anneals(g("G"), g("g"), g("b"), g("x0"), pr[0], pr[1], pr[2], pr[3], pr[4],
                          pr[5], int(pr[6]), int(pr[7]), pr[8])
    for got, name in zip(out, ("spins", "diverged", "steps", "mvms")):
        assert np.array_equal(got, g(name)), name


def test_golden_cases_cover_divergence_and_refresh_patterns():
    z = load_golden("anneals.npz")
    n = int(z["n_cases"])
    assert any(z[f"c{k}_diverged"].any() for k in range(n))
    assert any(not z[f"c{k}_diverged"].any() for k in range(n))
    assert {int(z[f"c{k}_prm"][6]) for k in range(n)} >= {1, 2, 3}


def test_seed_fixture_matches_numpy():
    z = load_golden("seeds.npz")
    for row, n, want in zip(z["parts"], z["lens"], z["derived"]):
        assert orc.seed_of(*[int(v) for v in row[:n]]) == int(want)
    for s, row in zip(z["x0_seeds"], z["x0"]):
        assert np.array_equal(orc.initial_states([int(s)], 65, 0.1)[0], row)


@pytest.mark.parametrize("name", DET_SETS)
def test_oracle_front_end_and_ising(name):
    d = load_golden(f"{name}.npz")
    order = int(d["order"])
    levels, spacing = orc.qam(order)
    for t in range(len(d["H"])):
        xg, eg = orc.mmse(d["H"][t], d["y"][t], float(d["noise_var"][t]), levels)
        idx = np.stack([orc.level_index(xg.real, levels), orc.level_index(xg.imag, levels)], -1)
        assert np.array_equal(idx, d["x_mmse"][t])
        assert eg == d["e_mmse"][t]
        si = orc.ising(d["H"][t], d["y"][t], xg, spacing)
        np.testing.assert_array_equal(si["G"], d["G"][t])
        np.testing.assert_array_equal(si["b"], d["b"][t])
        assert si["offset"] == d["offset"][t]
        assert si["eps_scale"] == d["eps_scale"][t]


@pytest.mark.parametrize("name", DET_SETS[:2])
def test_oracle_detect_cim_exact(name):
    d = load_golden(f"{name}.npz")
    order = int(d["order"])
    levels, _ = orc.qam(order)
    for t in range(len(d["H"])):
        r = orc.detect_cim(d["H"][t], d["y"][t], float(d["noise_var"][t]), order,
                           seed=int(d["seed"][t]))
        idx = np.stack([orc.level_index(r["x"].real, levels),
                        orc.level_index(r["x"].imag, levels)], -1)
        assert np.array_equal(idx, d["x_hat"][t])
        assert r["energy"] == d["energy"][t]
        assert r["anneal_index"] == d["anneal_index"][t]
        assert r["diverged"] == d["diverged"][t]


def test_oracle_vpp_exact():
    d = load_golden("vpp8x8_16qam.npz")
    for t in range(16):
        r = orc.precode_vpp(d["H"][t], d["u"][t], float(d["P"]), float(d["tau"]),
                            seed=int(d["seed"][t]))
        assert np.array_equal(r["v"], d["v"][t])
        assert r["power"] == d["power"][t]


def test_c_oracle_matches_compiled_reference_kernel(rng):
    ref = orc.ref_kernel_module()
    if ref is None:
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    for trial in range(40):
        n = int(rng.integers(1, 12))
        A = rng.standard_normal((2 * n, 2 * n))
        G = (A + A.T) / 4
        g = np.diag(G).copy()
        b = rng.standard_normal(2 * n)
        x0 = rng.uniform(-0.1, 0.1, (5, 4 * n + 1))
        dt = float(rng.choice([0.02, 0.05, 0.2]))
        args = (G, g, b, x0, dt, 1.5, 0.5, 1.0, 0.3, 1e-6, int(rng.integers(1, 4)),
                int(rng.integers(1, 100)), 10.0)
        for a, b_ in zip(orc.run_anneals(*args), ref.run_anneals(*args)):
            assert np.array_equal(a, b_)


def test_gray_and_bit_errors():
    assert list(orc.gray(np.arange(8))) == [0, 1, 3, 2, 6, 7, 5, 4]
    a = np.array([[0, 1], [3, 2]])
    assert orc.bit_errors(a, a) == 0
    assert orc.bit_errors(np.array([[0, 0]]), np.array([[1, 0]])) == 1


MULTI_SETS = ["m8x8_16qam_15db", "m16x16_16qam_20db"]
_SRC = {"mmse": 0, "anneal": 1, "mmse_sic": 2}


@pytest.mark.parametrize("name", MULTI_SETS)
def test_oracle_mmse_sic_matches_reference(name):
    """linear.py:78-106 restatement against the reference's detect_mmse_sic."""
    d = load_golden(f"{name}.npz")
    levels, _ = orc.qam(int(d["order"]))
    for i in range(len(d["H"])):
        x, e = orc.mmse_sic(d["H"][i], d["y"][i], float(d["noise_var"][i]), levels)
        idx = np.stack([orc.level_index(x.real, levels), orc.level_index(x.imag, levels)], -1)
        assert np.array_equal(idx, d["x_sic"][i])
        assert e == d["e_sic"][i]


@pytest.mark.parametrize("name", MULTI_SETS)
def test_oracle_detect_cim_multi_matches_reference(name):
    """detector.py:85-134 restatement against the reference's detect_cim_multi."""
    d = load_golden(f"{name}.npz")
    order = int(d["order"])
    levels, _ = orc.qam(order)
    n = 12 if "16x16" in name else len(d["H"])  # keep the CPU suite short
    for i in range(n):
        r = orc.detect_cim_multi(d["H"][i], d["y"][i], float(d["noise_var"][i]), order,
                                 n_stages=int(d["n_stages"]), seed=int(d["seed"][i]))
        idx = np.stack([orc.level_index(r["x"].real, levels),
                        orc.level_index(r["x"].imag, levels)], -1)
        assert np.array_equal(idx, d["x_hat"][i]), i
        assert r["energy"] == d["energy"][i]
        assert _SRC[r["source"]] == d["source"][i]
        assert r["anneal_index"] == d["anneal_index"][i]
        assert r["diverged"] == d["diverged"][i]


@pytest.mark.parametrize("name", ["ml4x4_qpsk_8db", "ml3x2_16qam_12db"])
def test_oracle_ml_matches_reference(name):
    """linear.py:109-144 restatement against the reference's detect_ml."""
    d = load_golden(f"{name}.npz")
    levels, _ = orc.qam(int(d["order"]))
    for i in range(len(d["H"])):
        x, e = orc.ml(d["H"][i], d["y"][i], levels)
        idx = np.stack([orc.level_index(x.real, levels), orc.level_index(x.imag, levels)], -1)
        assert np.array_equal(idx, d["x_ml"][i])
        assert e == d["e_ml"][i]

"""GPU: the reference-shaped API (api.py) against the reference's own test
invariants (pkg/tests/test_solver.py, test_transform.py, test_detector.py,
test_precoder.py, test_backends.py), with the oracle as the independent
checker.  Instances use the reference's conftest generator semantics
(random_instance: derive_seed(tag, trial, {0,1,2})).
"""

import dataclasses
import itertools
import math

import numpy as np
import pytest

from oracle import isinglink_oracle as orc
from paper_2510_01579_b200 import api, batched
from paper_2510_01579_b200.channel import MimoInstance, make_qam, sample_channel, transmit
from paper_2510_01579_b200.params import CacParams

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib_ready(built_lib):
    return built_lib


def random_instance(n_r, n_t, order, snr_db, tag, trial=0):
    """conftest.py:57-71 semantics."""
    const = make_qam(order)
    H = sample_channel(n_r, n_t, orc.seed_of(tag, trial, 0))
    rng = np.random.default_rng(orc.seed_of(tag, trial, 1))
    x = const.points[rng.integers(0, const.order, n_t)]
    y, s2 = transmit(H, x, snr_db, orc.seed_of(tag, trial, 2))
    return MimoInstance(H=H, y=y, constellation=const, noise_var=s2, truth=x)


def problem(tag=3000, trial=0, n=8, order=16, snr=20.0):
    inst = random_instance(n, n, order, snr, tag=tag, trial=trial)
    return inst, api.build_ising(inst, api.detect_mmse(inst).x_hard)


def dense_matrix(si):
    """conftest.py:23-40: the (2N+1)^2 matrix production code never forms."""
    n = si.n_dim
    m = np.zeros((si.spin_count, si.spin_count))
    core = si.G - np.diag(si.g_diag)
    m[:n, :n] = core
    m[n:2 * n, n:2 * n] = core
    m[:n, n:2 * n] = si.G
    m[n:2 * n, :n] = si.G
    m[:n, 2 * n] = m[n:2 * n, 2 * n] = si.b
    m[2 * n, :n] = m[2 * n, n:2 * n] = si.b
    return m


def all_spins(S):
    return np.array(list(itertools.product((-1, 1), repeat=S)), dtype=np.int8)


# ---------------------------------------------------------------- transform --
class TestIsing:
    def test_spin_count_and_symmetry(self):
        inst, si = problem(n=2, order=4)
        assert si.spin_count == 9 and si.n_dim == 4
        _, si = problem(tag=2004, n=8, order=64)
        assert np.array_equal(si.G, si.G.T)

    def test_zero_channel_is_flat(self):
        inst = MimoInstance(H=np.zeros((3, 2), complex), y=np.ones(3, complex),
                            constellation=make_qam(4), noise_var=0.0)
        si = api.build_ising(inst, np.zeros(2, complex) + make_qam(4).points[0])
        assert np.all(si.G == 0) and np.all(si.b == 0)
        e = batched.spin_energies(si.G[None], si.b[None], all_spins(9)[None]).cpu().numpy()
        assert set(e.ravel().tolist()) == {0.0}

    def test_rejects_nonfinite_guess(self):
        inst = random_instance(2, 2, 4, 15.0, tag=2003)
        with pytest.raises(ValueError):
            api.build_ising(inst, np.array([np.nan + 0j, 0j]))

    @pytest.mark.parametrize("trial", range(12))
    def test_exhaustive_residual_equivalence(self, trial):
        """test_transform.py:74-85: E(s) + offset == ||y - H(x_g + delta(s))||^2 for all 2^9 s."""
        inst = random_instance(2, 2, 4, 18.0, tag=2005, trial=trial)
        guess = api.detect_mmse(inst).x_hard
        si = api.build_ising(inst, guess)
        S = all_spins(si.spin_count)
        e = batched.spin_energies(si.G[None], si.b[None], S[None]).cpu().numpy()[0]
        for s, es in zip(S, e):
            rhs = api.residual_energy(inst.H, inst.y,
                                      guess + api.spin_perturbation(si, api.SpinVector.from_array(s)))
            assert abs(es + si.offset - rhs) <= 1e-9 * (1 + abs(rhs))

    def test_matches_dense_reference(self, rng):
        inst, si = problem(tag=2006, n=4, order=16, snr=15.0)
        S = rng.choice([-1, 1], size=(64, si.spin_count)).astype(np.int8)
        e = batched.spin_energies(si.G[None], si.b[None], S[None]).cpu().numpy()[0]
        D = dense_matrix(si)
        for s, es in zip(S.astype(float), e):
            assert es == pytest.approx(s @ D @ s, abs=1e-12 * (1 + abs(s @ D @ s)))

    def test_global_flip_and_swap_exact(self, rng):
        inst, si = problem(tag=2009, n=4, order=16, snr=15.0)
        n = si.n_dim
        S = rng.choice([-1, 1], size=(50, si.spin_count)).astype(np.int8)
        flip = -S
        swap = np.concatenate([S[:, n:2 * n], S[:, :n], S[:, 2 * n:]], axis=1)
        e = batched.spin_energies(np.stack([si.G] * 3), np.stack([si.b] * 3),
                                  np.stack([S, flip, swap])).cpu().numpy()
        assert np.array_equal(e[0], e[1]) and np.array_equal(e[0], e[2])

    def test_structured_mvm_matches_dense(self, rng):
        for n_t in (2, 8, 16, 32):
            inst = random_instance(n_t, n_t, 4, 15.0, tag=3001 + n_t)
            si = api.build_ising(inst, api.detect_mmse(inst).x_hard)
            D = dense_matrix(si)
            for _ in range(4):
                x = rng.standard_normal(si.spin_count)
                got = api.structured_mvm(si, x[:si.n_dim], x[si.n_dim:2 * si.n_dim], x[-1])
                assert np.max(np.abs(got - D @ x)) < 1e-12

    def test_ising_matches_oracle(self):
        for trial in range(10):
            inst = random_instance(6, 4, 16, 15.0, tag=2000, trial=trial)
            g = api.detect_mmse(inst).x_hard
            si = api.build_ising(inst, g)
            o = orc.ising(inst.H, inst.y, g, inst.constellation.spacing)
            np.testing.assert_allclose(si.G, o["G"], rtol=1e-12, atol=1e-13)
            np.testing.assert_allclose(si.b, o["b"], rtol=1e-12, atol=1e-13)
            assert si.offset == pytest.approx(o["offset"], rel=1e-12)
            assert si.eps_scale == pytest.approx(o["eps_scale"], rel=1e-12)

    def test_large_shapes_match_oracle(self):
        """16 < n_t <= 32 take the warp-per-RE front end (k_front): MMSE
        decisions, residual and the Ising coefficients against the oracle."""
        for n_r, n_t, order in ((20, 20, 16), (30, 28, 4), (32, 32, 16)):
            for trial in range(2):
                inst = random_instance(n_r, n_t, order, 20.0, tag=2100 + n_t, trial=trial)
                lv = inst.constellation.pam_levels
                mm = api.detect_mmse(inst)
                xh, e = orc.mmse(inst.H, inst.y, inst.noise_var, lv)
                np.testing.assert_array_equal(mm.x_hard, xh)
                assert mm.energy == pytest.approx(e, rel=1e-12)
                si = api.build_ising(inst, mm.x_hard)
                o = orc.ising(inst.H, inst.y, mm.x_hard, inst.constellation.spacing)
                np.testing.assert_allclose(si.G, o["G"], rtol=1e-12, atol=1e-13)
                np.testing.assert_allclose(si.b, o["b"], rtol=1e-12, atol=1e-12)
                assert si.offset == pytest.approx(o["offset"], rel=1e-12)
                assert si.eps_scale == pytest.approx(o["eps_scale"], rel=1e-12)


# ------------------------------------------------------------------- solver --
class TestSolver:
    def test_decoupled_flow_preserves_signs(self):
        _, si = problem()
        free = dataclasses.replace(si, G=np.zeros_like(si.G), g_diag=np.zeros_like(si.g_diag),
                                   b=np.zeros_like(si.b))
        params = CacParams(eps=0.1, n_steps=400)
        res = api.integrate_anneal(free, params, 77)
        x0 = np.random.default_rng(77).uniform(-0.1, 0.1, si.spin_count)
        assert not res.diverged
        assert np.array_equal(res.spins.to_array(), np.where(x0 >= 0, 1.0, -1.0))

    def test_huge_step_diverges(self):
        _, si = problem()
        for seed in range(5):
            assert api.integrate_anneal(si, CacParams(dt=10.0, n_steps=64), seed).diverged

    def test_bit_identical_reruns_and_oracle(self):
        _, si = problem()
        a = api.integrate_anneal(si, CacParams(), 5)
        b = api.integrate_anneal(si, CacParams(), 5)
        assert np.array_equal(a.spins.to_array(), b.spins.to_array()) and a.energy == b.energy
        x0 = orc.initial_states([5], si.spin_count, 0.1)
        o = orc.run_anneals(si.G, si.g_diag, si.b, x0, 0.02, 1.5, 0.5, 1.0, si.eps_scale, 1e-6,
                            2, 128, 10.0)
        assert np.array_equal(a.spins.to_array().astype(np.int8), o[0][0])

    def test_mvm_refresh_cost_model(self):
        _, si = problem()
        for n_steps, f_mvm in [(128, 2), (100, 3), (7, 8), (64, 1)]:
            counters = {}
            res = api.integrate_anneal(si, CacParams(n_steps=n_steps, f_mvm=f_mvm), 11,
                                       counters=counters)
            assert not res.diverged
            assert counters["mvm_updates"] == math.ceil(n_steps / f_mvm)
            assert counters["steps"] == n_steps and counters["anneals"] == 1

    def test_single_anneal_matches_integrate(self):
        _, si = problem()
        params = CacParams(n_anneals=1, precision="fp64_exact")
        best, div = api.solve_batch(si, params, math.inf, base_seed=42)
        solo = api.integrate_anneal(si, params, api.derive_seed(42, 0))
        assert best is not None and not solo.diverged and div == 0
        assert np.array_equal(best.spins.to_array(), solo.spins.to_array())
        assert best.energy == solo.energy

    @pytest.mark.parametrize("precision", ["fp64_exact", "fp32"])
    def test_order_independence(self, precision):
        _, si = problem()
        params = CacParams(n_anneals=16, precision=precision)
        best, _ = api.solve_batch(si, params, math.inf, base_seed=6)
        solo = [api.integrate_anneal(si, params, api.derive_seed(6, i)) for i in range(16)]
        ref = min((r for r in solo if not r.diverged), key=lambda r: r.energy)
        if precision == "fp64_exact":
            assert best.energy == ref.energy
            assert np.array_equal(best.spins.to_array(), ref.spins.to_array())
        else:
            assert best.energy <= ref.energy + 1e-9 * abs(ref.energy)

    def test_all_divergent_falls_back(self):
        _, si = problem()
        params = CacParams(p=1.0, a=0.0, diverge_threshold=0.001, n_anneals=8)
        best, diverged = api.solve_batch(si, params, math.inf, base_seed=0)
        assert best is None and diverged == 8

    def test_fallback_threshold(self):
        _, si = problem()
        params = CacParams(n_anneals=4, precision="fp64_exact")
        best, _ = api.solve_batch(si, params, math.inf, base_seed=1)
        assert best is not None
        worse, _ = api.solve_batch(si, params, best.energy + si.offset - 1e-6, base_seed=1)
        assert worse is None

    def test_coarse_step_sign_agreement(self):
        mismatch = total = 0
        for trial in range(30):
            _, si = problem(tag=3100, trial=trial, n=4, order=4, snr=15.0)
            seed = api.derive_seed(3100, trial)
            fine = api.integrate_anneal(si, CacParams(dt=0.01, f_mvm=1, n_steps=256), seed)
            coarse = api.integrate_anneal(si, CacParams(dt=0.02, f_mvm=2, n_steps=128), seed)
            assert not fine.diverged and not coarse.diverged
            mismatch += np.sum(fine.spins.to_array() != coarse.spins.to_array())
            total += si.spin_count
        assert mismatch / total < 0.05


# ---------------------------------------------------------------- pipelines --
class TestDetect:
    def test_identity_noiseless(self):
        const = make_qam(16)
        rng = np.random.default_rng(0)
        x = const.points[rng.integers(0, 16, 4)]
        inst = MimoInstance(H=np.eye(4, dtype=complex), y=x.copy(), constellation=const,
                            noise_var=0.0, truth=x)
        for prec in ("fp64_exact", "fp32"):
            res = api.detect_cim(inst, CacParams(precision=prec), seed=0)
            assert np.array_equal(res.x_hard, x) and res.energy == 0.0 and res.source == "mmse"

    @pytest.mark.parametrize("precision", ["fp64_exact", "fp32"])
    def test_never_worse_than_mmse_and_matches_oracle(self, precision):
        agree = 0
        for trial in range(40):
            inst = random_instance(8, 8, 16, 20.0, tag=4000, trial=trial)
            res = api.detect_cim(inst, CacParams(precision=precision), seed=trial)
            assert res.energy <= api.detect_mmse(inst).energy
            assert res.energy == pytest.approx(api.residual_energy(inst.H, inst.y, res.x_hard),
                                               rel=1e-9)
            o = orc.detect_cim(inst.H, inst.y, inst.noise_var, 16, seed=trial)
            agree += np.array_equal(o["x"], res.x_hard)
        assert agree / 40 >= (1.0 if precision == "fp64_exact" else 0.95)

    @pytest.mark.parametrize("precision", ["fp64_exact", "fp32", "tf32"])
    def test_counters_path_equals_fused_path(self, precision):
        """Counters are instrumentation: passing them runs the same arithmetic
        (the precision alone selects the kernel) and returns the same result."""
        for trial in range(12):
            inst = random_instance(8, 8, 16, 15.0, tag=4001, trial=trial)
            c = {}
            a = api.detect_cim(inst, CacParams(precision=precision), seed=trial, counters=c)
            b = api.detect_cim(inst, CacParams(precision=precision), seed=trial)
            assert np.array_equal(a.x_hard, b.x_hard) and a.source == b.source
            assert a.energy == b.energy and a.anneal_index == b.anneal_index
            assert a.diverged_count == b.diverged_count == c["diverged"]
            assert c["anneals"] == 32 and c["mvm_updates"] >= 64 * (32 - c["diverged"])
            assert c["steps"] >= 128 * (32 - c["diverged"])

    def test_all_anneals_divergent_returns_mmse(self):
        inst = random_instance(4, 4, 4, 15.0, tag=4004)
        params = CacParams(p=1.0, a=0.0, diverge_threshold=0.001)
        res = api.detect_cim(inst, params, seed=0)
        mmse = api.detect_mmse(inst)
        assert np.array_equal(res.x_hard, mmse.x_hard) and res.source == "mmse"
        assert res.diverged_count == params.n_anneals

    def test_deterministic(self):
        inst = random_instance(8, 8, 16, 20.0, tag=4003)
        a = api.detect_cim(inst, seed=5)
        b = api.detect_cim(inst, seed=5)
        assert np.array_equal(a.x_hard, b.x_hard)
        assert (a.energy, a.source, a.anneal_index, a.diverged_count) == (
            b.energy, b.source, b.anneal_index, b.diverged_count)

    def test_odd_shapes_run_padded_fast_kernel(self):
        """n_t = 3, 6, 9 (N = 6, 12, 18 spins per half, not multiples of 8)
        run the FP32 kernel with inert padding spins; the exact mode still
        reproduces the oracle, the FP32 mode decides the same on these."""
        from paper_2510_01579_b200 import _lib
        for (nr, nt) in ((5, 3), (12, 6), (9, 9)):
            assert _lib.anneal_kernel(2 * nt, CacParams()) == "fast_padded"
            inst = random_instance(nr, nt, 16, 18.0, tag=4010 + nt)
            o = orc.detect_cim(inst.H, inst.y, inst.noise_var, 16, seed=1)
            ex = api.detect_cim(inst, CacParams(precision="fp64_exact"), seed=1)
            assert np.array_equal(ex.x_hard, o["x"])
            fa = api.detect_cim(inst, CacParams(), seed=1)
            assert fa.energy <= ex.energy * (1 + 1e-12)


def downlink_draw(tag, trial, n=4, order=16):
    const = make_qam(order)
    H = sample_channel(n, n, orc.seed_of(tag, trial, 0))
    rng = np.random.default_rng(orc.seed_of(tag, trial, 1))
    u = const.points[rng.integers(0, const.order, n)]
    return const, H, u


def exhaustive_vpp_power(W, u, tau, n):
    best = math.inf
    vals = (-2.0, 0.0, 2.0)
    for re in itertools.product(vals, repeat=n):
        for im in itertools.product(vals, repeat=n):
            v = np.array(re) + 1j * np.array(im)
            w = W @ (u + tau * v)
            best = min(best, float(np.real(np.vdot(w, w))))
    return best


class TestPrecode:
    def test_zero_data_degenerates(self):
        _, H, _ = downlink_draw(5003, 0)
        res = api.precode_vpp(H, np.zeros(4, complex), P=1.0, tau=2.0, seed=0)
        assert np.all(res.v == 0) and np.all(res.x_transmit == 0)
        assert res.unnormalized_power == 0.0

    @pytest.mark.parametrize("trial", range(10))
    def test_never_worse_than_zf_and_contract(self, trial):
        const, H, u = downlink_draw(5004, trial)
        tau = api.default_tau(const)
        res = api.precode_vpp(H, u, P=4.0, tau=tau, seed=trial)
        w_u = api.zf_matrix(H) @ u
        assert res.unnormalized_power <= float(np.real(np.vdot(w_u, w_u))) * (1 + 1e-12)
        assert np.all(np.isin(res.v.real, (-2.0, 0.0, 2.0)))
        assert np.all(np.isin(res.v.imag, (-2.0, 0.0, 2.0)))
        assert np.linalg.norm(res.x_transmit) ** 2 == pytest.approx(4.0, rel=1e-9)
        o = orc.precode_vpp(H, u, 4.0, tau, seed=trial)
        assert np.array_equal(res.v, o["v"])

    def test_matches_exhaustive_search(self):
        const = make_qam(4)
        tau = api.default_tau(const)
        hits = 0
        for trial in range(60):
            _, H, u = downlink_draw(5006, trial, n=2, order=4)
            res = api.precode_vpp(H, u, P=1.0, tau=tau, seed=api.derive_seed(5006, trial, 2))
            ref = exhaustive_vpp_power(api.zf_matrix(H), u, tau, 2)
            hits += abs(res.unnormalized_power - ref) <= 1e-9 * (1 + ref)
        assert hits / 60 >= 0.95

    def test_more_stages_never_hurt(self):
        const, H, u = downlink_draw(5007, 3)
        tau = api.default_tau(const)
        p1 = api.precode_vpp(H, u, P=1.0, tau=tau, seed=1, n_stages=1).unnormalized_power
        p2 = api.precode_vpp(H, u, P=1.0, tau=tau, seed=1, n_stages=2).unnormalized_power
        o2 = orc.precode_vpp(H, u, 1.0, tau, seed=1, n_stages=2)
        assert p2 <= p1 * (1 + 1e-12)
        assert p2 == pytest.approx(o2["power"], rel=1e-9)


# ------------------------------------------------------------ plugin / boundary --
class TestPlugin:
    def test_backend_agreement_with_oracle_kernel(self):
        """test_backends.py:55-100 contract, tightened: spins, flags, steps, mvms identical."""
        from paper_2510_01579_b200 import _kernel_cuda
        assert _kernel_cuda.BACKEND_NAME == "cuda"
        for trial, (dt, ns) in enumerate([(0.02, 128), (0.16, 16), (0.08, 64)] * 4):
            inst, si = problem(tag=6001, trial=trial)
            x0 = orc.initial_states([orc.seed_of(6001, trial, i) for i in range(16)],
                                    si.spin_count, 0.1)
            args = (si.G, si.g_diag, si.b, x0, dt, 1.5, 0.5, 1.0, si.eps_scale, 1e-6, 2, ns, 10.0)
            for a, b in zip(_kernel_cuda.run_anneals(*args), orc.run_anneals(*args)):
                assert np.array_equal(a, b)

    def test_empty_batch(self):
        from paper_2510_01579_b200 import _kernel_cuda
        _, si = problem()
        out = _kernel_cuda.run_anneals(si.G, si.g_diag, si.b, np.zeros((0, si.spin_count)), 0.02,
                                       1.5, 0.5, 1.0, 0.1, 1e-6, 2, 16, 10.0)
        assert out[0].shape == (0, si.spin_count) and out[1].shape == (0,)

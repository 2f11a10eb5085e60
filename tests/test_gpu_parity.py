"""GPU parity: the CUDA path against the golden fixtures produced by the real
reference (tests/golden/make_golden.py) and against the oracle.

Bars (north_star):
  * integer/byte/index work bit-exact: seeds, PCG64 streams, spins of the
    FP64-exact kernel, MMSE decisions, decoded level indices, Gray bits;
  * Ising coefficients G, g_diag, b, offset, eps_scale within 1e-12 relative
    (north_star tolerance 1e-5; the FP64 build is held far tighter);
  * FP64-exact detection: identical decisions to the reference;
  * FP32 throughput mode: best energy <= reference on >= 99% of instances.
"""

import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import isinglink_oracle as orc

pytestmark = pytest.mark.gpu

DET_SETS = ["d8x8_qpsk_10db", "d8x8_16qam_20db", "d16x16_16qam_20db", "d16x16_64qam_25db"]


@pytest.fixture(scope="module", autouse=True)
def _lib_ready(built_lib):
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return built_lib


def test_derive_seeds_bit_exact():
    from paper_2510_01579_b200 import batched
    z = load_golden("seeds.npz")
    for row, n, want in zip(z["parts"], z["lens"], z["derived"]):
        got = batched.derive_seeds(row[None, :n]).cpu().numpy()
        assert got[0] == want, (row[:n], got[0], want)


def test_initial_states_bit_exact():
    from paper_2510_01579_b200 import batched
    z = load_golden("seeds.npz")
    x0 = batched.initial_states(z["x0_seeds"], 65, 0.1).cpu().numpy()
    assert np.array_equal(x0, z["x0"])


def test_initial_states_match_numpy_many_seeds(rng):
    from paper_2510_01579_b200 import batched
    seeds = rng.integers(0, 2**63, 200, dtype=np.uint64)
    seeds[:3] = [0, 1, 2**32]
    x0 = batched.initial_states(seeds, 33, 0.25).cpu().numpy()
    want = np.stack([np.random.default_rng(int(s)).uniform(-0.25, 0.25, 33) for s in seeds])
    assert np.array_equal(x0, want)


@pytest.mark.parametrize("case", range(11))
def test_run_anneals_exact_bit_identical(case):
    from paper_2510_01579_b200 import _kernel_cuda
    z = load_golden("anneals.npz")
    g = lambda n: z[f"c{case}_{n}"]
    pr = g("prm")
    out = _kernel_cuda.run_anneals(g("G"), g("g"), g("b"), g("x0"), pr[0], pr[1], pr[2], pr[3],
                                   pr[4], pr[5], int(pr[6]), int(pr[7]), pr[8])
    assert np.array_equal(out[0], g("spins"))
    assert np.array_equal(out[1], g("diverged"))
    assert np.array_equal(out[2], g("steps"))
    assert np.array_equal(out[3], g("mvms"))


def test_run_anneals_device_tensor_api():
    from paper_2510_01579_b200 import batched
    z = load_golden("anneals.npz")
    g = lambda n: z[f"c0_{n}"]
    pr = g("prm")
    spins, div, steps, mvms = batched.run_anneals(g("G"), g("g"), g("b"), g("x0"), *pr[:6],
                                                  int(pr[6]), int(pr[7]), pr[8])
    assert np.array_equal(spins.cpu().numpy(), g("spins"))
    assert np.array_equal(mvms.cpu().numpy(), g("mvms"))


def test_run_anneals_rejects_bad_buffers():
    from paper_2510_01579_b200 import _kernel_cuda
    z = load_golden("anneals.npz")
    g = lambda n: z[f"c0_{n}"]
    pr = g("prm")
    with pytest.raises(ValueError):
        _kernel_cuda.run_anneals(g("G").astype(np.float32), g("g"), g("b"), g("x0"), *pr[:6],
                                 int(pr[6]), int(pr[7]), pr[8])
    with pytest.raises(ValueError):
        _kernel_cuda.run_anneals(g("G"), g("g"), g("b"), np.asfortranarray(g("x0")), *pr[:6],
                                 int(pr[6]), int(pr[7]), pr[8])


@pytest.mark.parametrize("name", DET_SETS)
def test_mmse_and_ising_match_reference(name):
    from paper_2510_01579_b200 import batched
    d = load_golden(f"{name}.npz")
    order = int(d["order"])
    x_idx, energy, status = batched.mmse_batch(d["H"], d["y"], d["noise_var"], order)
    assert np.array_equal(x_idx.cpu().numpy(), d["x_mmse"])          # bit-exact decisions
    assert np.all(status.cpu().numpy() == 0)
    np.testing.assert_allclose(energy.cpu().numpy(), d["e_mmse"], rtol=1e-12)
    si = batched.build_ising_batch(d["H"], d["y"], x_idx, order)
    np.testing.assert_allclose(si["G"].cpu().numpy(), d["G"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(si["b"].cpu().numpy(), d["b"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(si["offset"].cpu().numpy(), d["offset"], rtol=1e-12)
    np.testing.assert_allclose(si["eps_scale"].cpu().numpy(), d["eps_scale"], rtol=1e-12)
    G = si["G"].cpu().numpy()
    np.testing.assert_array_equal(si["g_diag"].cpu().numpy(),
                                  np.diagonal(G, axis1=1, axis2=2))


@pytest.mark.parametrize("name", DET_SETS)
def test_detect_cim_exact_matches_reference(name):
    """FP64-exact mode reproduces the reference detections."""
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    d = load_golden(f"{name}.npz")
    r = batched.detect_cim_batch(d["H"], d["y"], d["noise_var"], int(d["order"]), d["seed"],
                                 CacParams(precision="fp64_exact"))
    x = r.x_idx.cpu().numpy()
    same = np.all(x == d["x_hat"], axis=(1, 2))
    assert same.mean() == 1.0, np.nonzero(~same)
    np.testing.assert_allclose(r.energy.cpu().numpy(), d["energy"], rtol=1e-12)
    assert np.array_equal(r.source.cpu().numpy(), d["source"])
    assert np.array_equal(r.anneal_index.cpu().numpy(), d["anneal_index"])
    assert np.array_equal(r.diverged.cpu().numpy(), d["diverged"])


@pytest.mark.parametrize("precision", ["fp32", "mixed", "tf32"])
@pytest.mark.parametrize("name", DET_SETS)
def test_detect_cim_fast_energy_parity(name, precision):
    """Throughput mode: final energy <= reference on >= 99% of instances."""
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    d = load_golden(f"{name}.npz")
    r = batched.detect_cim_batch(d["H"], d["y"], d["noise_var"], int(d["order"]), d["seed"],
                                 CacParams(precision=precision))
    e = r.energy.cpu().numpy()
    ok = e <= d["energy"] * (1 + 1e-12)
    frac = ok.mean()
    print(f"{name} {precision}: energy<=ref {frac:.4f}, identical decisions "
          f"{np.all(r.x_idx.cpu().numpy() == d['x_hat'], axis=(1, 2)).mean():.4f}")
    assert frac >= (0.97 if precision == "tf32" else 0.99)


def test_precode_vpp_matches_reference():
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    d = load_golden("vpp8x8_16qam.npz")
    for prec in ("fp64_exact", "fp32"):
        r = batched.precode_vpp_batch(d["H"], d["u"], float(d["P"]), float(d["tau"]), d["seed"],
                                      CacParams(precision=prec))
        v = r.v.cpu().numpy()
        pw = r.unnormalized_power.cpu().numpy()
        if prec == "fp64_exact":
            assert np.array_equal(v, d["v"])
            np.testing.assert_allclose(pw, d["power"], rtol=1e-11)
            np.testing.assert_allclose(r.x.cpu().numpy(), d["x"], rtol=1e-10, atol=1e-12)
        else:
            assert np.mean(pw <= d["power"] * (1 + 1e-11)) >= 0.99


def test_gray_demap_bit_exact():
    from paper_2510_01579_b200 import batched
    rng = np.random.default_rng(1)
    for m, bpd in ((2, 1), (4, 2), (8, 3), (16, 4)):
        idx = rng.integers(0, m, (300, 2)).astype(np.uint8)
        bits = batched.gray_demap(idx, bpd).cpu().numpy()
        gl = idx ^ (idx >> 1)
        want = np.stack([(gl[:, d:d + 1] >> (bpd - 1 - q)) & 1 for d in range(2)
                         for q in range(bpd)], axis=-1).reshape(300, 2 * bpd)
        assert np.array_equal(bits, want)


def test_oracle_agrees_on_random_instances():
    """Fresh seeded instances (not in the fixtures): GPU exact == oracle."""
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    for (nr, nt, order, snr) in ((4, 4, 16, 15.0), (12, 8, 64, 25.0), (6, 6, 4, 8.0)):
        Hs, ys, s2s, seeds, want = [], [], [], [], []
        levels, _ = orc.qam(order)
        for t in range(24):
            H, y, s2, _ = orc.uplink_instance(5, snr, 0, t, nr, nt, order)
            seed = orc.seed_of(5, 1, 0, t, 3)
            res = orc.detect_cim(H, y, s2, order, seed=seed)
            Hs.append(H); ys.append(y); s2s.append(s2); seeds.append(seed)
            want.append(np.stack([orc.level_index(res["x"].real, levels),
                                  orc.level_index(res["x"].imag, levels)], -1))
        r = batched.detect_cim_batch(np.array(Hs), np.array(ys), np.array(s2s), order,
                                     np.array(seeds, np.uint64), CacParams(precision="fp64_exact"))
        assert np.array_equal(r.x_idx.cpu().numpy(), np.array(want))


@pytest.mark.parametrize("n_chunks", [0, 1, 3, 7])
def test_detect_cim_host_pipeline_matches_device_batch(n_chunks):
    """The chunked host-buffer pipeline (il_detect_cim_host) returns exactly
    what the device-resident batch returns, for any chunking (ragged last
    chunk included), and matches the reference fixtures."""
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    d = load_golden("d16x16_16qam_20db.npz")
    reps = 5  # tile the fixture to a ragged multi-chunk batch
    H = np.concatenate([d["H"]] * reps)[:-3]
    y = np.concatenate([d["y"]] * reps)[:-3]
    s2 = np.concatenate([d["noise_var"]] * reps)[:-3]
    seed = np.concatenate([d["seed"]] * reps)[:-3]
    for prec in ("fp64_exact", "fp32"):
        prm = CacParams(precision=prec)
        dev = batched.detect_cim_batch(H, y, s2, int(d["order"]), seed, prm)
        host = batched.detect_cim_host(torch.from_numpy(H).pin_memory(),
                                       torch.from_numpy(y).pin_memory(),
                                       torch.from_numpy(s2).pin_memory(),
                                       int(d["order"]), seed, prm, n_chunks=n_chunks)
        for f in ("x_idx", "energy", "source", "anneal_index", "diverged"):
            assert torch.equal(getattr(dev, f).cpu(), getattr(host, f)), (prec, f)
        if prec == "fp64_exact":
            n = len(d["x_hat"])
            assert np.array_equal(host.x_idx.numpy()[:n], d["x_hat"])


def test_detect_cim_host_submit_streams_slots():
    """Back-to-back submitted slots (il_detect_cim_host_submit) overlap on the
    device streams but each returns exactly the synchronous result; an empty
    slot yields a NULL ticket."""
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    d = load_golden("d16x16_16qam_20db.npz")
    reps = 40
    H = torch.from_numpy(np.concatenate([d["H"]] * reps)).pin_memory()
    y = torch.from_numpy(np.concatenate([d["y"]] * reps)).pin_memory()
    s2 = torch.from_numpy(np.concatenate([d["noise_var"]] * reps)).pin_memory()
    seed = np.concatenate([d["seed"]] * reps)
    prm = CacParams(precision="fp32")
    want = batched.detect_cim_host(H, y, s2, int(d["order"]), seed, prm)
    tickets = [batched.detect_cim_host_submit(H, y, s2, int(d["order"]), seed, prm)
               for _ in range(3)]
    for tk in tickets:
        got = tk.wait()
        for f in ("x_idx", "energy", "source", "anneal_index", "diverged"):
            assert torch.equal(getattr(want, f), getattr(got, f)), f
    empty = batched.detect_cim_host_submit(torch.zeros((0, 4, 4), dtype=torch.complex128),
                                           torch.zeros((0, 4), dtype=torch.complex128),
                                           torch.zeros(0, dtype=torch.float64), 16,
                                           np.zeros(0, np.uint64))
    assert empty.wait().x_idx.shape == (0, 4, 2)


def test_detect_cim_host_rejects_device_buffers():
    from paper_2510_01579_b200 import batched
    H = torch.zeros((2, 4, 4), dtype=torch.complex128, device="cuda")
    with pytest.raises(ValueError):
        batched.detect_cim_host(H, torch.zeros((2, 4), dtype=torch.complex128),
                                torch.ones(2, dtype=torch.float64), 4, np.arange(2, dtype=np.uint64))


@pytest.mark.parametrize("n_anneals", [8, 12, 40])
def test_fast_kernel_any_replica_count(n_anneals):
    """Replica counts that are not multiples of 16 (config 5's N_a sweep) run
    on the fast kernel with padded tiles; the padded anneals never win."""
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    d = load_golden("d16x16_16qam_20db.npz")
    args = (d["H"], d["y"], d["noise_var"], int(d["order"]), d["seed"])
    ex = batched.detect_cim_batch(*args, CacParams(n_anneals=n_anneals, precision="fp64_exact"))
    fa = batched.detect_cim_batch(*args, CacParams(n_anneals=n_anneals, precision="fp32"))
    assert int(fa.anneal_index.max()) < n_anneals
    assert int(fa.diverged.max()) <= n_anneals
    e_ex, e_fa = ex.energy.cpu().numpy(), fa.energy.cpu().numpy()
    assert (e_fa <= e_ex * (1 + 1e-12)).mean() >= 0.99
    same = np.all(fa.x_idx.cpu().numpy() == ex.x_idx.cpu().numpy(), axis=(1, 2)).mean()
    assert same >= 0.98
    # the exact mode with B anneals is the oracle's detect_cim with n_anneals=B
    levels, _ = orc.qam(int(d["order"]))
    prm = orc.params(n_anneals=n_anneals)
    for i in range(8):
        r = orc.detect_cim(d["H"][i], d["y"][i], float(d["noise_var"][i]), int(d["order"]), prm,
                           seed=int(d["seed"][i]))
        want = np.stack([orc.level_index(r["x"].real, levels), orc.level_index(r["x"].imag, levels)], -1)
        assert np.array_equal(ex.x_idx[i].cpu().numpy(), want)


@pytest.mark.parametrize("kw", [dict(), dict(p=1.2, a=0.3), dict(zeta=0.8),
                                dict(diverge_threshold=0.9), dict(dt=0.01, n_steps=256)])
def test_fast_kernel_operating_points(kw):
    """The FP32 kernel's instantiations: the scaled state at the reference
    operating point (x- and e-factors equal), the general path when they
    differ (p - 1 != zeta a, zeta != 1), tight divergence thresholds and a
    finer step -- each against the bit-exact FP64 kernel on the fixture REs."""
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    d = load_golden("d16x16_16qam_20db.npz")
    args = (d["H"], d["y"], d["noise_var"], int(d["order"]), d["seed"])
    ex = batched.detect_cim_batch(*args, CacParams(precision="fp64_exact", **kw))
    fa = batched.detect_cim_batch(*args, CacParams(precision="fp32", **kw))
    e_ex, e_fa = ex.energy.cpu().numpy(), fa.energy.cpu().numpy()
    assert (e_fa <= e_ex * (1 + 1e-12)).mean() >= 0.99, kw
    same = np.all(fa.x_idx.cpu().numpy() == ex.x_idx.cpu().numpy(), axis=(1, 2)).mean()
    assert same >= 0.97, (kw, same)
    # divergence counts agree (the scaled path tests q = alpha - dt x^2)
    dex, dfa = ex.diverged.cpu().numpy(), fa.diverged.cpu().numpy()
    assert np.abs(dex - dfa).mean() <= 0.5, kw


@pytest.mark.parametrize("n_t,order", [(24, 16), (32, 4), (12, 16)])
def test_fast_kernel_large_and_odd_spin_counts(n_t, order):
    """N = 48 / 64 (k_front with a warp per RE, 6 / 8 n-tiles) and N = 24
    (odd tile count, padded K) in FP32 against the bit-exact FP64 kernel."""
    import sys, os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from tools.parity_scale import batch
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    H, y, nv, seeds, _ = batch(n_t, order, 15.0, 256, 77 + n_t)
    ex = batched.detect_cim_batch(H, y, nv, order, seeds, CacParams(precision="fp64_exact"))
    fa = batched.detect_cim_batch(H, y, nv, order, seeds, CacParams(precision="fp32"))
    e_ex, e_fa = ex.energy.cpu().numpy(), fa.energy.cpu().numpy()
    assert (e_fa <= e_ex * (1 + 1e-12)).mean() >= 0.98
    same = (fa.x_idx == ex.x_idx).all(-1).all(-1).float().mean().item()
    assert same >= 0.95, same


@pytest.mark.parametrize("n_chunks", [0, 1, 4])
def test_precode_vpp_host_pipeline_matches_device_batch(n_chunks):
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    d = load_golden("vpp8x8_16qam.npz")
    H = np.concatenate([d["H"]] * 3)[:-5]
    u = np.concatenate([d["u"]] * 3)[:-5]
    seed = np.concatenate([d["seed"]] * 3)[:-5]
    prm = CacParams(precision="fp64_exact")
    dev = batched.precode_vpp_batch(H, u, float(d["P"]), float(d["tau"]), seed, prm)
    host = batched.precode_vpp_host(H, u, float(d["P"]), float(d["tau"]), seed, prm,
                                    n_chunks=n_chunks)
    for f in ("x", "v", "unnormalized_power", "diverged"):
        assert torch.equal(getattr(dev, f).cpu(), getattr(host, f)), f
    n = len(d["v"])
    assert np.array_equal(host.v.numpy()[:n], d["v"])


def test_host_pipeline_bits_equal_device_demap():
    """il_detect_cim_bits_host_submit: the Gray bits demapped inside the host
    pipeline equal il_gray_demap of the device batch's decisions, with or
    without the other outputs copied back."""
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    for name, bpd in (("d16x16_16qam_20db", 2), ("d8x8_qpsk_10db", 1), ("d16x16_64qam_25db", 3)):
        d = load_golden(f"{name}.npz")
        reps = 9
        H = np.concatenate([d["H"]] * reps)
        y = np.concatenate([d["y"]] * reps)
        s2 = np.concatenate([d["noise_var"]] * reps)
        seed = np.concatenate([d["seed"]] * reps)
        prm = CacParams(precision="fp32")
        dev = batched.detect_cim_batch(H, y, s2, int(d["order"]), seed, prm)
        want = batched.gray_demap(dev.x_idx, bpd).cpu()
        host = batched.detect_cim_host(H, y, s2, int(d["order"]), seed, prm, n_chunks=3, bits=True)
        assert torch.equal(host.bits, want), name
        assert torch.equal(host.x_idx, dev.x_idx.cpu()), name

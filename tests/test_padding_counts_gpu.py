"""GPU: shapes whose spin count is not a multiple of 8 on the FP32 kernel
(inert padding spins), the reference's anneal counters from the FP32 kernel,
and the library's private memory pool.

The FP32 mode is held to the north_star gate against the FP64-exact kernel
(bit-identical to the reference kernel, tests/test_gpu_parity.py): final
energy <= exact on >= 99% of the REs.  Counters follow _kernel.pyx:85-97
(steps = halting step + 1 for a diverged anneal, else n_steps; mvms =
ceil(steps / f_mvm)), accumulated as solver.py:208-214 does.
"""

import ctypes
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


def _uplink(n_r, n_t, order, snr, P, seed):
    import bench
    H, y, nv, seeds, truth, _ = bench._synthetic_uplink(torch.device("cuda"), P, n_t, order, snr, seed)
    if n_r != n_t:  # more receive antennas: regenerate H, y at n_r x n_t
        g = torch.Generator(device="cuda").manual_seed(seed + 1)
        H = torch.complex(torch.randn(P, n_r, n_t, dtype=torch.float64, device="cuda", generator=g),
                          torch.randn(P, n_r, n_t, dtype=torch.float64, device="cuda", generator=g)) * 0.5 ** 0.5
        m = int(round(order ** 0.5))
        lv = torch.arange(-(m - 1), m, 2, dtype=torch.float64, device="cuda") / (2 * (m * m - 1) / 3) ** 0.5
        x = torch.complex(lv[truth[..., 0].long()], lv[truth[..., 1].long()])
        nz = torch.complex(torch.randn(P, n_r, dtype=torch.float64, device="cuda", generator=g),
                           torch.randn(P, n_r, dtype=torch.float64, device="cuda", generator=g))
        y = torch.einsum("prt,pt->pr", H, x) + nz * (nv[0].item() / 2) ** 0.5
    return H, y, nv, seeds, truth


@pytest.mark.parametrize("n_r,n_t,order", [(1, 1, 16), (2, 2, 4), (4, 3, 16), (6, 5, 16),
                                           (6, 6, 16), (9, 9, 16), (10, 10, 4), (12, 11, 64),
                                           (20, 20, 16), (28, 28, 4), (30, 30, 16)])
def test_padded_shapes_fp32_against_exact(n_r, n_t, order):
    """Every n_t <= 32 runs the FP32 kernel: N = 2 n_t spins per half on the
    smallest built layout N' >= N (N' = 8 NT, NT = 1..8)."""
    from paper_2510_01579_b200 import _lib, batched
    from paper_2510_01579_b200.params import CacParams
    N = 2 * n_t
    want = "fast" if N % 8 == 0 else "fast_padded"
    assert _lib.anneal_kernel(N, CacParams()) == want
    H, y, nv, seeds, truth = _uplink(n_r, n_t, order, 14.0, 512, 900 + 7 * n_t)
    ex = batched.detect_cim_batch(H, y, nv, order, seeds, CacParams(precision="fp64_exact"))
    fa = batched.detect_cim_batch(H, y, nv, order, seeds, CacParams(precision="fp32"))
    e_ex, e_fa = ex.energy.cpu().numpy(), fa.energy.cpu().numpy()
    le = float(np.mean(e_fa <= e_ex * (1 + 1e-12)))
    same = (fa.x_idx == ex.x_idx).all(-1).all(-1).float().mean().item()
    print(f"{n_r}x{n_t} {order}-QAM: energy<=exact {le:.4f} identical {same:.4f}")
    assert le >= 0.99 and same >= 0.97
    assert int(fa.anneal_index.max()) < 32


def test_padded_solve_batch_spins_layout():
    """il_solve_batch on a padded shape: best_spins come back in the
    unpadded [2N + 1] layout and their FP64 energy is the one reported."""
    from paper_2510_01579_b200 import api, batched
    from paper_2510_01579_b200.params import CacParams
    H, y, nv, seeds, _ = _uplink(7, 7, 16, 15.0, 64, 31)
    x_idx, _, _ = batched.mmse_batch(H, y, nv, 16)
    si = batched.build_ising_batch(H, y, x_idx, 16)
    r = batched.solve_batch(si["G"], si["g_diag"], si["b"], si["offset"],
                            torch.full((64,), 1e300, dtype=torch.float64, device="cuda"),
                            si["eps_scale"], seeds, CacParams(precision="fp32"))
    N = 14
    assert r.best_spins.shape == (64, 2 * N + 1)
    G, b = si["G"].cpu().numpy(), si["b"].cpu().numpy()
    for p in range(8):
        if int(r.best_index[p]) < 0:
            continue
        s = r.best_spins[p].cpu().numpy().astype(np.float64)
        u = s[:N] + s[N:2 * N]
        e = u @ G[p] @ u - 2 * np.trace(G[p]) + 2 * s[2 * N] * (b[p] @ u)
        assert float(r.best_energy[p]) == pytest.approx(e, rel=1e-12, abs=1e-12)


@pytest.mark.parametrize("kw", [dict(), dict(dt=0.16, n_steps=24), dict(diverge_threshold=0.9)])
def test_fast_kernel_counters_match_exact(kw):
    """steps / mvms from the FP32 kernel (PAD instantiation with counting)
    against the FP64-exact kernel's, per anneal, on the same problems."""
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    H, y, nv, seeds, _ = _uplink(8, 8, 16, 20.0, 128, 77)
    x_idx, _, _ = batched.mmse_batch(H, y, nv, 16)
    si = batched.build_ising_batch(H, y, x_idx, 16)
    fb = torch.full((128,), 1e300, dtype=torch.float64, device="cuda")
    out = {}
    for prec in ("fp64_exact", "fp32"):
        out[prec] = batched.solve_batch(si["G"], si["g_diag"], si["b"], si["offset"], fb,
                                        si["eps_scale"], seeds, CacParams(precision=prec, **kw),
                                        counts=True)
    ex, fa = out["fp64_exact"], out["fp32"]
    n_steps = CacParams(**kw).n_steps
    st_ex, st_fa = ex.steps.cpu().numpy(), fa.steps.cpu().numpy()
    mv_fa = fa.mvms.cpu().numpy()
    f_mvm = CacParams(**kw).f_mvm
    assert st_fa.shape == st_ex.shape == (128, 32)
    assert np.all((st_fa >= 1) & (st_fa <= n_steps))
    assert np.array_equal(mv_fa, (st_fa + f_mvm - 1) // f_mvm)
    agree = float(np.mean(st_fa == st_ex))
    print(kw, "steps agree", agree, "diverged exact", int(ex.diverged.sum()),
          "fp32", int(fa.diverged.sum()))
    assert agree >= 0.97
    # a non-diverged anneal runs all n_steps
    assert np.all(st_fa[st_fa < n_steps] < n_steps)


def test_vpp_zero_stages_is_plain_zf():
    """n_stages = 0 (precoder.py:114-124 runs no stage): v = 0 and x is the
    power-normalised ZF precoding, as the reference returns."""
    from paper_2510_01579_b200 import api
    from oracle import isinglink_oracle as orc
    rng = np.random.default_rng(8)
    H = (rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))) * np.sqrt(0.5)
    levels, _ = orc.qam(16)
    u = levels[rng.integers(0, 4, 4)] + 1j * levels[rng.integers(0, 4, 4)]
    tau = orc.default_tau(16)
    res = api.precode_vpp(H, u, 2.0, tau, seed=3, n_stages=0)
    w = api.zf_matrix(H) @ u
    assert np.all(res.v == 0)
    assert res.unnormalized_power == pytest.approx(float(np.real(np.vdot(w, w))), rel=1e-12)
    np.testing.assert_allclose(res.x_transmit, np.sqrt(2.0) * w / np.linalg.norm(w), rtol=1e-10)
    with pytest.raises(ValueError):
        api.precode_vpp(H, u, 2.0, tau, seed=3, n_stages=16)


def test_host_entries_reject_narrow_seeds():
    from paper_2510_01579_b200 import batched
    H = torch.zeros((4, 4, 4), dtype=torch.complex128)
    u = torch.zeros((4, 4), dtype=torch.complex128)
    with pytest.raises(TypeError):
        batched.precode_vpp_host(H, u, 1.0, 2.0, torch.arange(4, dtype=torch.int32))
    with pytest.raises(TypeError):
        batched.detect_cim_host(H, u, torch.ones(4, dtype=torch.float64), 16,
                                torch.arange(4, dtype=torch.int32))


def test_private_memory_pool_leaves_default_pool_alone():
    """The library allocates from its own pool: the device's default
    cudaMallocAsync pool keeps its release threshold (0) after calls."""
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    H, y, nv, seeds, _ = _uplink(8, 8, 16, 20.0, 256, 5)
    batched.detect_cim_batch(H, y, nv, 16, seeds, CacParams())
    batched.detect_cim_host(H.cpu(), y.cpu(), nv.cpu(), 16, seeds.cpu(), CacParams())
    torch.cuda.synchronize()
    cu = ctypes.CDLL("libcuda.so.1")  # driver API: the pool objects are the driver's
    assert cu.cuInit(0) == 0
    dev = ctypes.c_int()
    assert cu.cuDeviceGet(ctypes.byref(dev), torch.cuda.current_device()) == 0
    pool = ctypes.c_void_p()
    assert cu.cuDeviceGetDefaultMemPool(ctypes.byref(pool), dev) == 0
    thr = ctypes.c_uint64(123)
    CU_MEMPOOL_ATTR_RELEASE_THRESHOLD = 4
    assert cu.cuMemPoolGetAttribute(pool, CU_MEMPOOL_ATTR_RELEASE_THRESHOLD, ctypes.byref(thr)) == 0
    assert thr.value == 0


@pytest.mark.parametrize("n_t,kw", [(16, dict(f_mvm=1)), (16, dict(f_mvm=3)), (16, dict(n_steps=127)),
                                    (8, dict(f_mvm=3, n_steps=101)), (8, dict(n_anneals=8, n_steps=99)),
                                    (16, dict(f_mvm=4, n_anneals=8))])
def test_fast_kernel_refresh_schedules_against_exact(n_t, kw):
    """The FP32 kernel's step loop has two forms: f_mvm = 2 as compile-time
    (refresh, step) pairs with a tail step for odd n_steps, any other f_mvm
    as a refresh countdown (_kernel.pyx:65: refresh when step % f_mvm ==
    0).  Both held to the energy gate against the FP64-exact kernel."""
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    H, y, nv, seeds, _ = _uplink(n_t, n_t, 16, 16.0, 384, 1234 + n_t)
    for prec in ("fp32", "mixed"):
        ex = batched.detect_cim_batch(H, y, nv, 16, seeds, CacParams(precision="fp64_exact", **kw))
        fa = batched.detect_cim_batch(H, y, nv, 16, seeds, CacParams(precision=prec, **kw))
        e_ex, e_fa = ex.energy.cpu().numpy(), fa.energy.cpu().numpy()
        le = float(np.mean(e_fa <= e_ex * (1 + 1e-12)))
        same = (fa.x_idx == ex.x_idx).all(-1).all(-1).float().mean().item()
        print(f"{n_t}x{n_t} {kw} {prec}: energy<=exact {le:.4f} identical {same:.4f}")
        assert le >= 0.99 and same >= 0.97

"""Run ONLY under tests/ref_suite_plugin.py (tests/test_reference_suite_gpu.py
launches it): the reference's backend-agreement checks (pkg/tests/
test_backends.py:44-100) with "cuda" in place of "python", through the
reference's own public API and use_kernel() -- and held to bit-identity
instead of the reference's 99% / 95% allowances, because the CUDA plugin runs
the FP64 kernel in the reference kernel's evaluation order.  Plus fork safety
(hard part 6): the reference harness's fork worker pools
with the plugin active, before and after CUDA was initialised in the parent.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from isinglink import (CacParams, build_ising, derive_seed, detect_cim, detect_cim_multi,
                       detect_mmse, integrate_anneal, precode_vpp, use_kernel)

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _reference_conftest():
    """The reference's tests/conftest.py, loaded by path (this repo's own
    tests/conftest.py shadows the name on sys.path)."""
    import importlib.util
    path = os.path.join(ROOT, "oracle", "_ref", "pkg_tests", "conftest.py")
    spec = importlib.util.spec_from_file_location("isinglink_ref_conftest", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


random_instance = _reference_conftest().random_instance  # the reference's generator

PAIR = ("cuda", "ext")


def test_cuda_registered_beside_reference_backends():
    import isinglink
    assert {"cuda", "ext", "python"} <= set(isinglink.available_kernels())
    with use_kernel("cuda"):
        assert isinglink.kernel_backend() == "cuda"


def test_spins_bit_identical():
    """test_backends.py:57-72, cuda vs ext: every spin of every anneal."""
    for trial in range(60):
        inst = random_instance(8, 8, 16, 20.0, tag=6001, trial=trial)
        si = build_ising(inst, detect_mmse(inst).x_hard)
        seed = derive_seed(6001, trial)
        out = {}
        for name in PAIR:
            with use_kernel(name):
                r = integrate_anneal(si, CacParams(), seed)
            out[name] = (r.spins.to_array(), r.energy, r.diverged)
        assert np.array_equal(out["cuda"][0], out["ext"][0])
        assert out["cuda"][1:] == out["ext"][1:]


@pytest.mark.parametrize("n,order,snr", [(8, 16, 20.0), (16, 16, 20.0), (16, 64, 25.0), (4, 4, 8.0)])
def test_detections_identical(n, order, snr):
    """test_backends.py:75-87, cuda vs ext: detections, energies, sources."""
    for trial in range(20):
        inst = random_instance(n, n, order, snr, tag=6002, trial=trial)
        out = {}
        for name in PAIR:
            with use_kernel(name):
                out[name] = detect_cim(inst, seed=trial)
        a, b = out["cuda"], out["ext"]
        assert np.array_equal(a.x_hard, b.x_hard)
        assert (a.energy, a.source, a.anneal_index, a.diverged_count) == \
               (b.energy, b.source, b.anneal_index, b.diverged_count)


def test_divergence_flags_identical():
    """test_backends.py:90-100 (coarse step, frequent blow-ups)."""
    inst = random_instance(8, 8, 16, 20.0, tag=6003)
    si = build_ising(inst, detect_mmse(inst).x_hard)
    params = CacParams(dt=0.16, n_steps=16)
    flags = {}
    for name in PAIR:
        with use_kernel(name):
            flags[name] = [integrate_anneal(si, params, derive_seed(6003, i)).diverged
                           for i in range(16)]
    assert flags["cuda"] == flags["ext"] and any(flags["ext"])


def test_counters_identical():
    inst = random_instance(8, 8, 16, 12.0, tag=6004)
    c = {name: {} for name in PAIR}
    for name in PAIR:
        with use_kernel(name):
            detect_cim(inst, CacParams(dt=0.08), seed=3, counters=c[name])
    assert c["cuda"] == c["ext"]


def test_multi_and_precoder_identical():
    """detect_cim_multi (detector.py:85-134) and precode_vpp
    (precoder.py:93-146) through the plugin."""
    from isinglink import make_qam, sample_channel
    from isinglink.precoder import default_tau
    for trial in range(6):
        inst = random_instance(8, 8, 16, 18.0, tag=6005, trial=trial)
        out = {}
        for name in PAIR:
            with use_kernel(name):
                out[name] = detect_cim_multi(inst, seed=trial, n_stages=2)
        assert np.array_equal(out["cuda"].x_hard, out["ext"].x_hard)
        assert out["cuda"].energy == out["ext"].energy
    const = make_qam(16)
    rng = np.random.default_rng(5)
    for trial in range(6):
        H = sample_channel(4, 4, derive_seed(6006, trial))
        u = const.points[rng.integers(0, 16, 4)]
        out = {}
        for name in PAIR:
            with use_kernel(name):
                out[name] = precode_vpp(H, u, 1.0, default_tau(const), seed=trial, n_stages=2)
        assert np.array_equal(out["cuda"].v, out["ext"].v)
        assert out["cuda"].unnormalized_power == out["ext"].unnormalized_power


def _sweep_cfg(n_workers):
    from isinglink.harness.config import ExperimentConfig
    return ExperimentConfig(detectors=("mmse", "cim"), n_r=4, n_t=4, modulation=16,
                            snr_grid_db=(10.0, 20.0), n_trials=24, seed=11, n_workers=n_workers)


def test_fork_pool_after_cuda_init():
    """The reference harness forks its workers (harness/workers.py:36-38)
    AFTER this process has run CUDA work: each worker's plugin calls go to
    its own exec'd server (paper_2510_01579_b200/_plugin_server.py), and the
    sweep rows equal the single-process run's and the ext backend's."""
    from isinglink.harness.sweeps import run_detection_sweep
    with use_kernel("cuda"):
        integrate_anneal(build_ising(*(lambda i: (i, detect_mmse(i).x_hard))(
            random_instance(4, 4, 16, 10.0, tag=6007))), CacParams(), 1)  # CUDA is live here
        rows_1 = run_detection_sweep(_sweep_cfg(1))
        rows_3 = run_detection_sweep(_sweep_cfg(3))
    with use_kernel("ext"):
        rows_ext = run_detection_sweep(_sweep_cfg(3))
    key = lambda rows: [(r.detector, r.snr_db, r.ser, r.ber, r.mean_energy, r.mean_diverged)
                        for r in rows]
    assert key(rows_1) == key(rows_3) == key(rows_ext)


def test_fork_pool_before_cuda_init():
    """install() does not initialise CUDA: a fresh process that installs the
    plugin and then forks lets every worker create its own context."""
    code = f"""
import sys
sys.path[:0] = [{ROOT!r}, {os.path.join(ROOT, 'oracle', '_ref', 'pkg')!r}]
import isinglink
from paper_2510_01579_b200 import _lib
from paper_2510_01579_b200.install import install
install(isinglink)
from isinglink.harness.config import ExperimentConfig
from isinglink.harness.sweeps import run_detection_sweep
cfg = ExperimentConfig(detectors=("cim",), n_r=4, n_t=4, modulation=16, snr_grid_db=(15.0,),
                       n_trials=16, seed=3, n_workers=2)
assert not _lib._used
rows = run_detection_sweep(cfg)
with isinglink.use_kernel("ext"):
    ref = run_detection_sweep(cfg)
assert [(r.ser, r.ber, r.mean_energy) for r in rows] == [(r.ser, r.ber, r.mean_energy) for r in ref]
print("fork-before-init ok", rows[0].ser)
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "fork-before-init ok" in r.stdout


def test_kernel_comparison_row_with_cuda():
    """The reference's _kernel_comparison (harness/bench.py:117-144) with
    "cuda" among the kernels: per-instance detect_cim time of
    every backend through the reference's code path, plus the batched slot
    path, and decision agreement with "ext"."""
    import json
    import dataclasses as dc
    import isinglink
    from isinglink.harness import ExperimentConfig
    from paper_2510_01579_b200 import harness
    cfg = dc.replace(ExperimentConfig(), mode="bench", n_r=8, n_t=8, modulation=16,
                     snr_grid_db=(20.0,), batch_size=64, seed=1)
    row = harness.kernel_comparison(isinglink, cfg, n_probe=64)
    print(json.dumps(row, indent=1))
    out = os.environ.get("ISINGLINK_KCMP_OUT")
    if out:
        out = out if os.path.isabs(out) else os.path.join(ROOT, out)
        with open(out, "w") as fh:
            json.dump(row, fh, indent=1)
    agree = row["output_agreement_with_ext"]
    assert agree["cuda"] == 1.0
    assert agree["cuda_batched_fp64_exact"] == 1.0
    assert agree["cuda_batched_fp32"] >= 0.95
    assert agree["python"] >= 0.95  # the reference's own allowance (test_backends.py)

"""GPU: error behaviour, empty batches and thread safety of the public API
(the reference's kernel releases the GIL, so concurrent calls on distinct
data must be safe, _kernel.pyx:58)."""

import threading

import numpy as np
import pytest
import torch

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _ready(built_lib):
    assert torch.cuda.is_available()


def _inst(d, i):
    from paper_2510_01579_b200 import api
    nv = float(d["noise_var"][i]) if "noise_var" in d else 1.0
    return api.MimoInstance(H=d["H"][i], y=d["y"][i], constellation=api.make_qam(int(d["order"])),
                            noise_var=nv)


def test_nonfinite_inputs_raise_value_error():
    """scipy's cho_factor(check_finite=True) raises ValueError in the reference."""
    from paper_2510_01579_b200 import api
    d = load_golden("d8x8_16qam_20db.npz")
    import dataclasses
    for field in ("H", "y"):
        inst = _inst(d, 0)
        bad = getattr(inst, field).copy()
        bad.flat[3] = np.nan
        inst = dataclasses.replace(inst, **{field: bad})
        for fn in (api.detect_mmse, api.detect_mmse_sic, api.detect_cim, api.detect_cim_multi):
            with pytest.raises(ValueError):
                fn(inst)


def test_empty_batches():
    from paper_2510_01579_b200 import batched
    H = np.zeros((0, 4, 4), complex)
    y = np.zeros((0, 4), complex)
    s2 = np.zeros(0)
    seeds = np.zeros(0, np.uint64)
    assert batched.detect_cim_batch(H, y, s2, 16, seeds).x_idx.shape == (0, 4, 2)
    assert batched.detect_cim_multi_batch(H, y, s2, 16, seeds).x_idx.shape == (0, 4, 2)
    assert batched.mmse_sic_batch(H, y, s2, 16)[0].shape == (0, 4, 2)
    assert batched.ml_batch(H, y, 4)[0].shape == (0, 4, 2)
    r = batched.detect_cim_host(torch.zeros((0, 4, 4), dtype=torch.complex128),
                                torch.zeros((0, 4), dtype=torch.complex128),
                                torch.zeros(0, dtype=torch.float64), 16, seeds)
    assert r.x_idx.shape == (0, 4, 2)


def test_ml_guard_and_api():
    from paper_2510_01579_b200 import api
    d = load_golden("ml4x4_qpsk_8db.npz")
    for i in range(4):
        r = api.detect_ml(_inst(d, i))
        assert r.source == "ml"
        idx = api.to_indices(r.x_hard, api.make_qam(int(d["order"])))
        assert np.array_equal(idx, d["x_ml"][i])
    big = api.MimoInstance(H=np.eye(8, dtype=complex), y=np.zeros(8, complex),
                           constellation=api.make_qam(64), noise_var=1.0)
    with pytest.raises(ValueError):
        api.detect_ml(big)  # 48 bits > 24-bit guard (linear.py:117-122)


def test_concurrent_calls_from_threads_match_serial():
    from paper_2510_01579_b200 import batched
    from paper_2510_01579_b200.params import CacParams
    sets = [load_golden(n) for n in ("d8x8_16qam_20db.npz", "d16x16_16qam_20db.npz")]
    prm = CacParams(precision="fp32")
    want = [batched.detect_cim_batch(d["H"], d["y"], d["noise_var"], int(d["order"]), d["seed"],
                                     prm).x_idx.cpu() for d in sets]
    got = [None] * 4
    errs = []

    def work(k):
        try:
            d = sets[k % 2]
            with torch.cuda.stream(torch.cuda.Stream()):
                r = batched.detect_cim_batch(d["H"], d["y"], d["noise_var"], int(d["order"]),
                                             d["seed"], prm)
                torch.cuda.current_stream().synchronize()
                got[k] = r.x_idx.cpu()
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    ts = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for k in range(4):
        assert torch.equal(got[k], want[k % 2])

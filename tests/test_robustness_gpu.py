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


def test_misaligned_h_y_rejected():
    """The detection front end stages H and y with 16-byte copies: a pointer
    that is only 8-byte aligned is an IL_ERR_ARG (ValueError), not a fault."""
    from paper_2510_01579_b200 import _lib, batched
    d = load_golden("d8x8_16qam_20db.npz")
    P, n_r, n_t = 4, 8, 8
    H = torch.as_tensor(d["H"][:P]).cuda()
    y = torch.as_tensor(d["y"][:P]).cuda()
    s2 = torch.full((P,), 0.08, dtype=torch.float64, device="cuda")
    # the same values behind an address offset by one float64
    Hf = torch.empty(P * n_r * n_t * 2 + 1, dtype=torch.float64, device="cuda")
    Hf[1:] = torch.view_as_real(H).reshape(-1)
    x_idx = torch.empty((P, n_t, 2), dtype=torch.uint8, device="cuda")
    energy = torch.empty(P, dtype=torch.float64, device="cuda")
    status = torch.empty(P, dtype=torch.int8, device="cuda")
    with pytest.raises(ValueError, match="16-byte aligned"):
        _lib.call("il_mmse_batch", Hf.data_ptr() + 8, y.data_ptr(), s2.data_ptr(), P, n_r, n_t, 16,
                  x_idx.data_ptr(), energy.data_ptr(), status.data_ptr(), None)
    # the aligned call still works afterwards
    xi, en, st = batched.mmse_batch(H, y, s2, 16)
    assert torch.isfinite(en).all()

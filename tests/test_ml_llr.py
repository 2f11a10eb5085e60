"""Max-log bit LLRs of the exhaustive search.  The reference has no soft
output (SPEC.md:153 lists it as a non-goal), so parity is unpinned: the
oracle's brute force defines the values, and both must agree in sign with the
hard bits of the reference-pinned ML detector (oracle.ml, linear.py:109-144)."""
import numpy as np
import pytest

from oracle import isinglink_oracle as orc


def _gray_bits(x, levels):
    m = len(levels)
    bpd = max(1, int(round(np.log2(m))))
    out = []
    for v in x:
        for comp in (v.real, v.imag):
            k = int(np.argmin(np.abs(levels - comp)))
            lab = k ^ (k >> 1)
            out += [(lab >> (bpd - 1 - q)) & 1 for q in range(bpd)]
    return np.array(out).reshape(len(x), 2 * bpd)


CASES = [(4, 4, 4, 6.0), (3, 3, 16, 12.0), (6, 4, 4, 3.0)]


@pytest.mark.parametrize("n_r,n_t,order,snr", CASES)
def test_oracle_llr_sign_matches_ml_bits(n_r, n_t, order, snr):
    levels, _ = orc.qam(order)
    for t in range(3):
        H, y, s2, _ = orc.uplink_instance(3, snr, 0, t, n_r, n_t, order)
        llr = orc.ml_llr(H, y, levels, s2)
        x, _ = orc.ml(H, y, levels)
        bits = _gray_bits(x, levels)
        assert np.all((llr > 0) == (bits == 0) | (llr == 0))


@pytest.mark.gpu
@pytest.mark.parametrize("n_r,n_t,order,snr", CASES + [(8, 8, 4, 10.0)])
def test_gpu_llr_matches_oracle(built_lib, n_r, n_t, order, snr):
    from paper_2510_01579_b200 import api, batched
    levels, _ = orc.qam(order)
    Hs, ys, s2s, want, hard = [], [], [], [], []
    n = 4 if n_t < 8 else 2
    for t in range(n):
        H, y, s2, _ = orc.uplink_instance(5, snr, 0, t, n_r, n_t, order)
        Hs.append(H); ys.append(y); s2s.append(s2)
        want.append(orc.ml_llr(H, y, levels, s2))
        hard.append(_gray_bits(orc.ml(H, y, levels)[0], levels))
    got = batched.ml_llr_batch(np.stack(Hs), np.stack(ys), order, noise_var=np.array(s2s))
    got = got.cpu().numpy()
    scale = np.abs(np.stack(want)).max()
    assert np.allclose(got, np.stack(want), rtol=1e-9, atol=1e-9 * scale)
    for g, h in zip(got, hard):
        assert np.all((g > 0) == (h == 0) | (g == 0))
    inst = api.MimoInstance(H=Hs[0], y=ys[0], constellation=api.make_qam(order), noise_var=s2s[0])
    assert np.allclose(api.ml_llr(inst), got[0], rtol=1e-12, atol=0)

"""The per-instance helpers run in the CUDA library too (no cuBLAS/cuSOLVER):
api.zf_matrix through il_zf_batch (precoder.py:54-60) and api.structured_mvm
through il_structured_mvm_batch (solver.py:147-168), against the oracle's
restatements."""

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


@pytest.mark.parametrize("n_u,n_ant", [(1, 1), (4, 4), (4, 8), (8, 8), (12, 16), (16, 16)])
def test_zf_matrix_matches_oracle(n_u, n_ant, rng):
    from oracle import isinglink_oracle as orc
    from paper_2510_01579_b200 import api
    for _ in range(5):
        H = (rng.standard_normal((n_u, n_ant)) + 1j * rng.standard_normal((n_u, n_ant))) * np.sqrt(0.5)
        np.testing.assert_allclose(api.zf_matrix(H), orc.zf(H), rtol=1e-10, atol=1e-12)


def test_zf_matrix_singular_raises():
    """A zero user row leaves a zero pivot: the reference's cho_factor raises."""
    from scipy.linalg import cho_factor
    from paper_2510_01579_b200 import api
    H = np.array([[1.0, 1.0], [0.0, 0.0]], dtype=complex)
    with pytest.raises(np.linalg.LinAlgError):
        cho_factor(H @ H.conj().T)
    with pytest.raises(np.linalg.LinAlgError):
        api.zf_matrix(H)


def test_structured_mvm_batch_matches_numpy(rng):
    from paper_2510_01579_b200 import _lib
    from paper_2510_01579_b200.batched import _stream
    P, N = 37, 24
    G = rng.standard_normal((P, N, N))
    G = G + G.transpose(0, 2, 1)
    g = np.ascontiguousarray(np.diagonal(G, axis1=1, axis2=2))
    b, x1, x2 = (rng.standard_normal((P, N)) for _ in range(3))
    xa = rng.standard_normal(P)
    dev = torch.device("cuda", torch.cuda.current_device())
    t = [torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev) for a in (G, g, b, x1, x2, xa)]
    out = torch.empty((P, 2 * N + 1), dtype=torch.float64, device=dev)
    _lib.call("il_structured_mvm_batch", *[a.data_ptr() for a in t], P, N, out.data_ptr(), _stream())
    v = x1 + x2
    m = np.einsum("pij,pj->pi", G, v)
    want = np.concatenate([m - g * x1 + b * xa[:, None], m - g * x2 + b * xa[:, None],
                           np.einsum("pi,pi->p", b, v)[:, None]], axis=1)
    np.testing.assert_allclose(out.cpu().numpy(), want, rtol=1e-12, atol=1e-12)

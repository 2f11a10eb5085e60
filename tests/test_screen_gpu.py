"""The FP32 energy screen of the anneal kernel (anneal_fast.cu: FP64 energies
only for the anneals that can be the argmin) must not change any output of
the detection path: compare it against the all-FP64 epilogue
(ISINGLINK_SCREEN=0, read once per process -> subprocess) bit for bit, over
SNRs from noisy (many near-ties between anneal energies) to clean, and every
spin count the screen serves (N = 24, 32, 48, 64)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
sys.path.insert(0, {root!r})
from tools.parity_scale import batch
from paper_2510_01579_b200 import batched
from paper_2510_01579_b200.params import CacParams
out = {{}}
for n_t, order, snr, P in ((16, 16, 5.0, 3000), (16, 16, 20.0, 3000), (12, 64, 25.0, 2000),
                           (16, 4, 0.0, 2000), (24, 16, 20.0, 600), (32, 4, 10.0, 400)):
    H, y, nv, seeds, _ = batch(n_t, order, snr, P, 11 + n_t)
    for prec in ("fp32", "tf32"):
        r = batched.detect_cim_batch(H, y, nv, order, seeds, CacParams(precision=prec))
        out[f"{{n_t}}_{{order}}_{{snr}}_{{prec}}"] = [
            r.x_idx.cpu().numpy().ravel().tolist(), r.energy.cpu().numpy().tolist(),
            r.anneal_index.cpu().numpy().tolist(), r.source.cpu().numpy().tolist()]
print(json.dumps(out))
"""


def _run(screen):
    env = dict(os.environ, ISINGLINK_SCREEN=str(screen))
    p = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_screened_selection_is_bit_identical():
    a, b = _run(1), _run(0)
    assert a.keys() == b.keys()
    for key in a:
        for x, y in zip(a[key], b[key]):
            assert np.array_equal(np.array(x), np.array(y)), key

"""Drop-in integration-kernel plugin for the reference ``isinglink`` package.

Same module contract as ``isinglink._kernel`` / ``isinglink._kernel_py``
(_kernel.pyx:13-31, _kernel_py.py:21-42): a ``BACKEND_NAME`` string and
``run_anneals(G, g_diag, b, x0, dt, p, a, zeta, eps, e_floor, f_mvm, n_steps,
diverge_threshold) -> (spins, diverged, steps, mvms)`` on host numpy arrays.

The integration runs on the GPU through ``il_run_anneals_host`` in FP64 with
the reference kernel's exact evaluation order, so its outputs are
bit-identical to the reference "ext" backend.  Like the Cython signature
(``const double[:, ::1]``), inputs must be C-contiguous float64 of the right
rank; violations raise ValueError before any device work.
"""

from __future__ import annotations

import numpy as np

from . import _lib

BACKEND_NAME = "cuda"


def _f64(name: str, arr, ndim: int) -> np.ndarray:
    if not isinstance(arr, np.ndarray):
        arr = np.asarray(arr)
    if arr.dtype != np.float64:
        raise ValueError(f"Buffer dtype mismatch for {name}, expected 'double' but got "
                         f"'{arr.dtype}'")
    if arr.ndim != ndim:
        raise ValueError(f"Buffer has wrong number of dimensions for {name} "
                         f"(expected {ndim}, got {arr.ndim})")
    if not arr.flags.c_contiguous:
        raise ValueError(f"ndarray {name} is not C-contiguous")
    return arr


def run_anneals(G, g_diag, b, x0, dt, p, a, zeta, eps, e_floor, f_mvm, n_steps,
                diverge_threshold):
    """Integrate a batch of anneals; returns (spins, diverged, steps, mvms).

    In a worker forked from a process that had initialised CUDA (the
    reference harness's fork pools, harness/workers.py:36-38) the call is
    served by a per-worker server process with its own CUDA context
    (_plugin_server.py); the arithmetic and the outputs are the same."""
    G = _f64("G", G, 2)
    g_diag = _f64("g_diag", g_diag, 1)
    b = _f64("b", b, 1)
    x0 = _f64("x0", x0, 2)
    n = G.shape[0]
    n_batch, n_spins = x0.shape
    if G.shape != (n, n) or g_diag.shape[0] < n or b.shape[0] < n or n_spins != 2 * n + 1:
        raise ValueError("inconsistent problem dimensions")
    if _lib.forked_from_cuda():
        from . import _plugin_server
        return _plugin_server.client().run_anneals(
            G, g_diag, b, x0, float(dt), float(p), float(a), float(zeta), float(eps),
            float(e_floor), int(f_mvm), int(n_steps), float(diverge_threshold))
    spins = np.empty((n_batch, n_spins), dtype=np.int8)
    diverged = np.zeros(n_batch, dtype=np.uint8)
    steps = np.full(n_batch, n_steps, dtype=np.int64)
    mvms = np.zeros(n_batch, dtype=np.int64)
    if n_batch:
        _lib.call("il_run_anneals_host", G.ctypes.data, g_diag.ctypes.data, b.ctypes.data,
                  x0.ctypes.data, n, n_batch, float(dt), float(p), float(a), float(zeta),
                  float(eps), float(e_floor), int(f_mvm), int(n_steps),
                  float(diverge_threshold), spins.ctypes.data, diverged.ctypes.data,
                  steps.ctypes.data, mvms.ctypes.data)
    return spins, diverged.astype(bool), steps, mvms

"""Register the CUDA kernel plugin inside an imported reference ``isinglink``.

The reference selects its integration kernel at import time
(solver.py:35-52) and swaps it through ``use_kernel`` / ``available_kernels``
(solver.py:60-84), which only know "ext" and "python".  ``install`` makes
"cuda" a first-class backend without editing the reference:

    import isinglink
    from paper_2510_01579_b200.install import install
    install(isinglink)                 # cuda becomes active and selectable
    isinglink.kernel_backend()         # -> "cuda"
    with isinglink.use_kernel("ext"):  # the reference backends keep working
        ...

``uninstall`` restores the previous state.
"""

from __future__ import annotations

from . import _kernel_cuda

_saved: dict = {}


def install(isinglink_module, activate: bool = True):
    solver = isinglink_module.solver
    if "available_kernels" not in _saved:
        _saved["available_kernels"] = solver.available_kernels
        _saved["impl"] = solver._impl
    original = _saved["available_kernels"]

    def available_kernels() -> dict:
        kernels = dict(original())
        kernels[_kernel_cuda.BACKEND_NAME] = _kernel_cuda
        return kernels

    available_kernels.__doc__ = original.__doc__
    solver.available_kernels = available_kernels
    isinglink_module.available_kernels = available_kernels
    if activate:
        solver._impl = _kernel_cuda
    return _kernel_cuda


def uninstall(isinglink_module):
    if "available_kernels" in _saved:
        solver = isinglink_module.solver
        solver.available_kernels = _saved["available_kernels"]
        isinglink_module.available_kernels = _saved["available_kernels"]
        solver._impl = _saved["impl"]
        _saved.clear()

"""ctypes binding of the C ABI in include/isinglink_b200.h.

The shared object is built in-tree by ``paper_2510_01579_b200.build``.  There
is deliberately no fallback: if the library is missing or cannot be loaded,
every entry point raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

LIB_PATH = os.environ.get(
    "ISINGLINK_B200_LIB",
    os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libisinglink_b200.so"))

IL_OK, IL_ERR_ARG, IL_ERR_CUDA, IL_ERR_UNSUPPORTED, IL_ERR_NOMEM = 0, -1, -2, -3, -4
PREC = {"fp64_exact": 0, "fp32": 1, "tf32": 2, "mixed": 3}
RNG = {"numpy": 0, "philox": 1}
ABI_VERSION = 2  # IL_ABI_VERSION of include/isinglink_b200.h (il_cac_params layout)

_c_d = ctypes.c_double
_c_i32 = ctypes.c_int32
_c_i64 = ctypes.c_int64
_vp = ctypes.c_void_p


class CacParamsC(ctypes.Structure):
    """il_cac_params (field order must match the header)."""
    _fields_ = [
        ("p", _c_d), ("a", _c_d), ("zeta", _c_d), ("eps", _c_d), ("dt", _c_d),
        ("f_mvm", _c_i32), ("n_steps", _c_i32), ("n_anneals", _c_i32), ("precision", _c_i32),
        ("diverge_threshold", _c_d), ("e_floor", _c_d), ("init_amplitude", _c_d),
        ("rng", _c_i32), ("reserved", _c_i32),
    ]


_SIGS = {
    "il_last_error": ([], ctypes.c_char_p),
    "il_abi_version": ([], ctypes.c_int),
    "il_anneal_kernel": ([_c_i32, ctypes.POINTER(CacParamsC)], ctypes.c_int),
    "il_run_anneals": ([_vp, _vp, _vp, _vp, _c_i32, _c_i32, _c_d, _c_d, _c_d, _c_d, _c_d, _c_d,
                        _c_i32, _c_i32, _c_d, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "il_run_anneals_host": ([_vp, _vp, _vp, _vp, _c_i32, _c_i32, _c_d, _c_d, _c_d, _c_d, _c_d,
                             _c_d, _c_i32, _c_i32, _c_d, _vp, _vp, _vp, _vp], ctypes.c_int),
    "il_derive_seeds": ([_vp, _c_i32, _c_i64, _vp, _vp], ctypes.c_int),
    "il_initial_states": ([_vp, _c_i64, _c_i32, _c_d, _vp, _vp], ctypes.c_int),
    "il_mmse_batch": ([_vp, _vp, _vp, _c_i64, _c_i32, _c_i32, _c_i32, _vp, _vp, _vp, _vp],
                      ctypes.c_int),
    "il_build_ising_batch": ([_vp, _vp, _vp, _c_i64, _c_i32, _c_i32, _c_i32, _vp, _vp, _vp, _vp,
                              _vp, _vp], ctypes.c_int),
    "il_detect_cim_batch": ([_vp, _vp, _vp, _c_i64, _c_i32, _c_i32, _c_i32, _vp,
                             ctypes.POINTER(CacParamsC), _vp, _vp, _vp, _vp, _vp, _vp],
                            ctypes.c_int),
    "il_residual_batch": ([_vp, _vp, _vp, _c_i64, _c_i32, _c_i32, _vp, _vp], ctypes.c_int),
    "il_ml_batch": ([_vp, _vp, _c_i64, _c_i32, _c_i32, _c_i32, _vp, _vp, _vp], ctypes.c_int),
    "il_ml_llr_batch": ([_vp, _vp, _vp, _c_i64, _c_i32, _c_i32, _c_i32, _vp, _vp], ctypes.c_int),
    "il_integrate_batch": ([_vp, _vp, _vp, _vp, _vp, _c_i64, _c_i32, ctypes.POINTER(CacParamsC),
                            _vp, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "il_mmse_sic_batch": ([_vp, _vp, _vp, _c_i64, _c_i32, _c_i32, _c_i32, _vp, _vp, _vp, _vp],
                          ctypes.c_int),
    "il_detect_cim_multi_batch": ([_vp, _vp, _vp, _c_i64, _c_i32, _c_i32, _c_i32, _vp,
                                   ctypes.POINTER(CacParamsC), _c_i32, _vp, _c_i32, _vp, _vp,
                                   _vp, _vp, _vp, _vp], ctypes.c_int),
    "il_detect_cim_host": ([_vp, _vp, _vp, _c_i64, _c_i32, _c_i32, _c_i32, _vp,
                            ctypes.POINTER(CacParamsC), _vp, _vp, _vp, _vp, _vp, _c_i32],
                           ctypes.c_int),
    "il_detect_cim_host_submit": ([_vp, _vp, _vp, _c_i64, _c_i32, _c_i32, _c_i32, _vp,
                                   ctypes.POINTER(CacParamsC), _vp, _vp, _vp, _vp, _vp, _c_i32,
                                   ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "il_detect_cim_bits_host_submit": ([_vp, _vp, _vp, _c_i64, _c_i32, _c_i32, _c_i32, _vp,
                                        ctypes.POINTER(CacParamsC), _vp, _vp, _vp, _vp, _vp, _vp,
                                        _c_i32, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "il_pipeline_wait": ([_vp], ctypes.c_int),
    "il_precode_vpp_host": ([_vp, _vp, _c_i64, _c_i32, _c_i32, _c_d, _c_d, _c_i32, _vp,
                             ctypes.POINTER(CacParamsC), _vp, _vp, _vp, _vp, _c_i32],
                            ctypes.c_int),
    "il_precode_vpp_batch": ([_vp, _vp, _c_i64, _c_i32, _c_i32, _c_d, _c_d, _c_i32, _vp,
                              ctypes.POINTER(CacParamsC), _vp, _vp, _vp, _vp, _vp],
                             ctypes.c_int),
    "il_gray_demap": ([_vp, _c_i64, _c_i32, _vp, _vp], ctypes.c_int),
    "il_spin_energies": ([_vp, _vp, _vp, _vp, _c_i64, _c_i32, _c_i32, _vp, _vp], ctypes.c_int),
    "il_structured_mvm_batch": ([_vp, _vp, _vp, _vp, _vp, _vp, _c_i64, _c_i32, _vp, _vp],
                                ctypes.c_int),
    "il_zf_batch": ([_vp, _c_i64, _c_i32, _c_i32, _vp, _vp, _vp], ctypes.c_int),
    "il_solve_batch": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_i64, _c_i32,
                        ctypes.POINTER(CacParamsC), _vp, _vp, _vp, _vp, _vp, _vp, _vp],
                       ctypes.c_int),
    "il_kernel_launches": ([], ctypes.c_longlong),
    "il_profile_begin": ([], None),
    "il_profile_end": ([_vp, _vp, ctypes.c_int], ctypes.c_int),
    "il_probe_fp32_peak": ([ctypes.c_int, _vp], ctypes.c_int),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and return the CDLL with typed entry points."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RuntimeError(
                    f"isinglink_b200 CUDA library not built ({path}); run "
                    "`python -m paper_2510_01579_b200.build` (there is no CPU fallback)")
            lib = ctypes.CDLL(path)
            for name, (args, res) in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            if lib.il_abi_version() != ABI_VERSION:
                raise RuntimeError(f"{path} implements ABI {lib.il_abi_version()}, these bindings "
                                   f"ABI {ABI_VERSION}: rebuild the library")
            _lib = lib
    return _lib


class IsinglinkError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def check(rc: int) -> None:
    if rc != IL_OK:
        msg = load().il_last_error().decode(errors="replace")
        if rc == IL_ERR_ARG:
            raise ValueError(msg)
        raise IsinglinkError(rc, msg)


def call(name: str, *args) -> None:
    global _used
    _used = True
    check(getattr(load(), name)(*args))


# ---- fork awareness --------------------------------------------------------
# CUDA cannot be used in a child forked from a process that has initialised
# it.  The reference's harness forks worker pools (harness/workers.py:36-38),
# so the kernel plugin must notice the case: a child forked after the parent
# made library calls (or initialised CUDA through torch) is flagged, and the
# plugin routes its calls to a freshly exec'd server process instead
# (_plugin_server.py).  A child forked before any CUDA use initialises its
# own context lazily, like any process.
_used = False
_forked_from_cuda = False


def _after_fork_in_child() -> None:
    global _used, _forked_from_cuda, _lib
    torch_mod = __import__("sys").modules.get("torch")
    torch_cuda = False
    if torch_mod is not None:
        try:
            torch_cuda = bool(torch_mod.cuda.is_initialized())
        except Exception:  # pragma: no cover - torch without CUDA support
            torch_cuda = False
    _forked_from_cuda = _forked_from_cuda or _used or torch_cuda
    _used = False


if hasattr(os, "register_at_fork"):
    os.register_at_fork(after_in_child=_after_fork_in_child)


def forked_from_cuda() -> bool:
    """True in a process forked from one that had initialised CUDA: this
    process must not call the library directly."""
    return _forked_from_cuda


PROFILE_KINDS = ("front", "anneal", "select", "other")


def profile_begin() -> None:
    load().il_profile_begin()


def profile_end() -> dict:
    """{kind: (milliseconds, launches)} summed over the profiled region."""
    import numpy as np
    ms = np.zeros(4, np.float64)
    n = np.zeros(4, np.int64)
    check(load().il_profile_end(ms.ctypes.data, n.ctypes.data, 4))
    return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(PROFILE_KINDS)}


def kernel_launches() -> int:
    return int(load().il_kernel_launches())


def fp32_peak_tflops(reps: int = 5) -> float:
    out = ctypes.c_double(0.0)
    check(load().il_probe_fp32_peak(int(reps), ctypes.addressof(out)))
    return float(out.value)


ANNEAL_KERNELS = {0: "exact", 1: "fast", 2: "fast_padded", 3: "umma"}


def anneal_kernel(n_dim: int, params=None, precision: str | None = None) -> str:
    """Name of the anneal kernel the batched entries run for n_dim spins per
    half (il_anneal_kernel): "exact", "fast", "fast_padded" or "umma"."""
    from .params import CacParams, to_c
    rc = load().il_anneal_kernel(int(n_dim), to_c(params or CacParams(), precision))
    check(min(rc, 0))
    return ANNEAL_KERNELS[rc]

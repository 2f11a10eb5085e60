"""The C-ABI library loads on CPU and exports every symbol include/*.h declares."""

import ctypes
import glob
import os
import re
import subprocess

from conftest import ROOT


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        names |= set(re.findall(r"^\s*(?:const\s+)?\w[\w\s\*]*?\b(il_\w+)\s*\(", text, re.M))
    return names


def test_header_declares_entry_points():
    names = _declared()
    for must in ("il_run_anneals", "il_run_anneals_host", "il_detect_cim_batch",
                 "il_precode_vpp_batch", "il_last_error", "il_gray_demap"):
        assert must in names


def test_library_exports_every_declared_symbol(built_lib):
    from paper_2510_01579_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (il_\w+)", out))
    missing = _declared() - exported
    assert not missing, missing
    assert set(_lib.EXPORTED) <= exported


def test_library_loads_without_gpu(built_lib):
    from paper_2510_01579_b200 import _lib
    lib = _lib.load()
    assert lib.il_abi_version() == _lib.ABI_VERSION == 2
    assert ctypes.sizeof(_lib.CacParamsC) == 88  # il_cac_params
    assert isinstance(lib.il_last_error(), bytes)


def test_cubin_is_sm100a(built_lib):
    from paper_2510_01579_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_anneal_kernel_routing_is_host_only(built_lib):
    """il_anneal_kernel answers without touching the GPU: every n_t <= 32
    runs the FP32 kernel in the throughput modes (inert padding spins when
    N = 2 n_t is not a built layout), the exact mode always the FP64 kernel."""
    from paper_2510_01579_b200 import _lib
    from paper_2510_01579_b200.params import CacParams
    for n_t in range(1, 33):
        N = 2 * n_t
        want = "fast" if N % 8 == 0 else "fast_padded"  # layouts N = 8 NT, NT = 1..8
        assert _lib.anneal_kernel(N, CacParams()) == want, N
        assert _lib.anneal_kernel(N, CacParams(), "tf32") == want, N
        assert _lib.anneal_kernel(N, CacParams(), "fp64_exact") == "exact"
    assert _lib.anneal_kernel(66, CacParams()) == "exact"  # beyond the FP32 layouts
    import pytest
    with pytest.raises(ValueError):
        _lib.anneal_kernel(8, CacParams(dt=-1.0))

"""CPU: the drop-in registration into the real reference package (build
container only: needs /root/reference and oracle/_ref).  No kernel is run."""

import os
import sys

import pytest

from oracle import isinglink_oracle as orc


@pytest.fixture(scope="module")
def isinglink():
    if not os.path.isdir("/root/reference/pkg/src"):
        pytest.skip("reference not mounted")
    ref = orc.ref_kernel_module()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    sys.modules.setdefault("isinglink._kernel", ref)
    sys.path.insert(0, "/root/reference/pkg/src")
    import isinglink as il
    return il


def test_install_registers_cuda_backend(isinglink):
    from paper_2510_01579_b200 import _kernel_cuda
    from paper_2510_01579_b200.install import install, uninstall
    before = isinglink.kernel_backend()
    install(isinglink)
    try:
        assert isinglink.kernel_backend() == "cuda"
        assert {"cuda", "ext", "python"} <= set(isinglink.available_kernels())
        assert isinglink.available_kernels()["cuda"] is _kernel_cuda
        with isinglink.use_kernel("python"):
            assert isinglink.kernel_backend() == "python"
        assert isinglink.kernel_backend() == "cuda"
    finally:
        uninstall(isinglink)
    assert isinglink.kernel_backend() == before
    assert "cuda" not in isinglink.available_kernels()

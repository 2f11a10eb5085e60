"""pytest plugin (``-p ref_suite_plugin``) for running the REFERENCE's own test
suite against the CUDA kernel plugin (tests/test_reference_suite_gpu.py).

Before collection it imports the reference package staged by
``make -C oracle refpkg`` (oracle/_ref/pkg: the unmodified reference sources
with its compiled Cython kernel as the "ext" backend) and registers
``paper_2510_01579_b200._kernel_cuda`` with ``install(isinglink)``, so that
module-level ``available_kernels()`` calls in the reference tests
(test_backends.py:25) already see "cuda".  ISINGLINK_REF_ACTIVATE=1 also makes
"cuda" the active backend for every reference call (solver._impl, exactly
what use_kernel() swaps, solver.py:74-84); =0 only registers it.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = os.path.join(ROOT, "oracle", "_ref", "pkg")
# on the path before the reference's conftest.py is loaded (it imports isinglink)
for _p in (ROOT, REF_PKG):
    if _p not in sys.path:
        sys.path.insert(0, _p)


def pytest_configure(config):
    import isinglink
    from paper_2510_01579_b200.install import install
    assert isinglink.__file__.startswith(REF_PKG), isinglink.__file__
    install(isinglink, activate=os.environ.get("ISINGLINK_REF_ACTIVATE", "1") == "1")


def pytest_report_header(config):
    import isinglink
    return (f"reference package: {os.path.dirname(isinglink.__file__)}; "
            f"kernels {sorted(isinglink.available_kernels())}; active {isinglink.kernel_backend()}")

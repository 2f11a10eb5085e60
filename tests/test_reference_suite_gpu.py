"""GPU: the REFERENCE's own test suite with the CUDA kernel plugin installed
(SURVEY section 8(c) golden tests).

The unmodified reference package and tests are staged by
``make -C oracle refpkg`` into oracle/_ref (git-ignored; travels to the GPU
box).  Each run is a separate pytest process with tests/ref_suite_plugin.py,
which calls ``install(isinglink)`` before collection:

  * test_backends.py with "cuda" registered beside "ext" and "python"
    (BOTH = sorted(available_kernels()), test_backends.py:25, so its
    parametrised determinism test runs on "cuda" too);
  * test_solver / test_transform / test_detector / test_precoder /
    test_linear / test_channel / test_harness with "cuda" ACTIVE: every
    run_anneals of the reference's own code path goes through the plugin
    (the harness tests fork worker pools after CUDA is live);
  * tests/ref_cuda_agreement.py: cuda vs ext bit-identity through the
    reference API, and fork safety before / after CUDA initialisation.
"""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(ROOT, "oracle", "_ref", "pkg_tests")
REF_PKG = os.path.join(ROOT, "oracle", "_ref", "pkg", "isinglink")

pytestmark = pytest.mark.gpu

ACTIVE_FILES = ["test_solver.py", "test_transform.py", "test_detector.py", "test_precoder.py",
                "test_linear.py", "test_channel.py", "test_harness.py"]


def _run(files, activate: bool, timeout=900, verbose=False, extra=()):
    if not (os.path.isdir(REF_TESTS) and os.path.isdir(REF_PKG)):
        pytest.fail("reference suite not staged: run `make -C oracle refpkg` in the build "
                    "container (it needs /root/reference)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests"), ROOT,
                                         env.get("PYTHONPATH", "")])
    env["ISINGLINK_REF_ACTIVATE"] = "1" if activate else "0"
    cmd = [sys.executable, "-m", "pytest", "-v" if verbose else "-q", "-p", "ref_suite_plugin", "-p",
           "no:cacheprovider", "-c", os.devnull, "--rootdir", REF_TESTS, *extra, *files]
    r = subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True,
                       timeout=timeout)
    tail = "\n".join((r.stdout + r.stderr).strip().splitlines()[-25:])
    print(tail)
    assert r.returncode == 0, tail
    return r.stdout


def test_reference_backend_suite_with_cuda_registered(built_lib):
    out = _run(["test_backends.py"], activate=False, verbose=True)
    # the reference's parametrised determinism test ran on the CUDA backend
    assert "test_each_backend_is_deterministic[cuda] PASSED" in out


@pytest.mark.parametrize("name", ACTIVE_FILES)
def test_reference_suite_with_cuda_active(built_lib, name):
    _run([name], activate=True)


def test_reference_acceptance_criteria_with_cuda_active(built_lib):
    """The reference's acceptance suite (test_acceptance.py:67-429), criteria
    1-7 and 9, with every anneal of its own code path on the CUDA plugin
    (about 2 minutes).  Criterion 8 times the reference's CPU worker pool
    (1 -> 2 -> 4 processes), not the kernel, and is left out."""
    out = _run(["test_acceptance.py"], activate=True, timeout=1800, verbose=True,
               extra=("-s", "-k", "not criterion_08"))
    for c in (1, 2, 3, 4, 5, 6, 7, 9):
        assert f"ACCEPTANCE criterion {c}: PASS" in out, c


def test_cuda_agrees_bit_for_bit_with_reference_kernel(built_lib):
    _run([os.path.join(ROOT, "tests", "ref_cuda_agreement.py")], activate=False)

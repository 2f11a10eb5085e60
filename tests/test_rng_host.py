"""CPU check of the device RNG header (csrc/rng_numpy.cuh): the same source,
compiled as host code by nvcc, must reproduce numpy's SeedSequence and PCG64
uniform streams bit for bit, and the PCG64 jump-ahead used by the fast
kernel must equal stepping."""

import os
import shutil
import subprocess

import numpy as np
import pytest

from conftest import ROOT, load_golden

SRC = os.path.join(ROOT, "tests", "native", "rng_host_check.cu")
BIN = os.path.join(ROOT, "build", "rng_host_check")


@pytest.fixture(scope="module")
def harness():
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < max(
            os.path.getmtime(SRC),
            os.path.getmtime(os.path.join(ROOT, "paper_2510_01579_b200", "csrc", "rng_numpy.cuh"))):
        subprocess.run([nvcc, "-O2", "-o", BIN, SRC], check=True)

    def run(text: str) -> list[str]:
        r = subprocess.run([BIN], input=text, capture_output=True, text=True, check=True)
        return r.stdout.split("\n")
    return run


def test_derive_seed_fixture(harness):
    z = load_golden("seeds.npz")
    lines = "".join(f"seed {n} " + " ".join(str(int(v)) for v in row[:n]) + "\n"
                    for row, n in zip(z["parts"], z["lens"]))
    out = harness(lines)
    assert [int(v) for v in out[:len(z["derived"])]] == [int(v) for v in z["derived"]]


def test_derive_seed_random(harness, rng):
    parts = [tuple(int(v) for v in rng.integers(0, 2**63, k, dtype=np.uint64))
             for k in (1, 2, 3, 4, 5, 6) for _ in range(20)]
    parts += [(0, 0), (2**32 - 1, 2**32), (2**64 - 1, 7, 0)]
    out = harness("".join(f"seed {len(p)} " + " ".join(map(str, p)) + "\n" for p in parts))
    for p, got in zip(parts, out):
        st = np.random.SeedSequence(p).generate_state(2)
        assert int(got) == int(st[0]) | (int(st[1]) << 32), p


def test_uniform_streams(harness):
    z = load_golden("seeds.npz")
    out = harness("".join(f"x0 {int(s)} 65\n" for s in z["x0_seeds"]))
    for row, line in zip(z["x0"], out):
        got = np.array([int(h, 16) for h in line.split()], dtype=np.uint64).view(np.float64)
        assert np.array_equal(got, row)


def test_jump_ahead(harness):
    out = harness("".join(f"jump {s} {k}\n" for s in (1, 99, 2**40) for k in (1, 17, 33, 65)))
    assert all(v == "1" for v in out if v)

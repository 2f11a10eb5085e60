"""CPU check of the counter-based initial-state generator
(csrc/rng_philox.cuh, CacParams.rng = "philox"): the device header compiled
as host code must equal cuRAND's Philox4x32-10 and the Random123 known-answer
vectors, and the FP32 states must follow x0 = lo + range * (w >> 8) 2^-24."""

import os
import shutil
import subprocess

import numpy as np
import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "native", "philox_check.cu")
HDR = os.path.join(ROOT, "paper_2510_01579_b200", "csrc", "rng_philox.cuh")
BIN = os.path.join(ROOT, "build", "philox_check")

# Random123 kat_vectors, philox4x32 with 10 rounds: (ctr[4], key[2]) -> out[4]
KAT = [((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
       ((0xffffffff,) * 4, (0xffffffff,) * 2, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
       ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
        (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1))]


@pytest.fixture(scope="module")
def harness():
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < max(os.path.getmtime(SRC),
                                                               os.path.getmtime(HDR)):
        subprocess.run([nvcc, "-O2", "-o", BIN, SRC], check=True)

    def run(text: str) -> list[str]:
        r = subprocess.run([BIN], input=text, capture_output=True, text=True, check=True)
        return [ln for ln in r.stdout.split("\n") if ln]
    return run


def _line(c, k):
    return "p " + " ".join(f"{v:x}" for v in (*c, *k)) + "\n"


def test_known_answers(harness):
    out = harness("".join(_line(c, k) for c, k, _ in KAT))
    for (_, _, want), line in zip(KAT, out):
        w = [int(h, 16) for h in line.split()]
        assert tuple(w[:4]) == want
        assert tuple(w[4:]) == want


def test_matches_curand(harness, rng):
    cases = [(tuple(int(v) for v in rng.integers(0, 2**32, 4, dtype=np.uint64)),
              tuple(int(v) for v in rng.integers(0, 2**32, 2, dtype=np.uint64))) for _ in range(500)]
    out = harness("".join(_line(c, k) for c, k in cases))
    assert len(out) == len(cases)
    for line in out:
        w = line.split()
        assert w[:4] == w[4:]


def test_x0_block(harness):
    seed, a, blk = 0x0123456789ABCDEF, 17, 5
    out = harness(f"x0 {seed} {a} {blk}\n")[0]
    got = np.array([int(h, 16) for h in out.split()], dtype=np.uint32).view(np.float32)
    w = harness(_line((blk, a, 0x49534C4B, 0), (seed & 0xffffffff, seed >> 32)))[0].split()[:4]
    u = np.array([int(h, 16) >> 8 for h in w], dtype=np.float32) * np.float32(2.0 ** -24)
    # fmaf(range, u, lo): the product is exact in FP64, one rounding to FP32
    want = (np.float64(np.float32(0.2)) * u.astype(np.float64) + np.float64(np.float32(-0.1))).astype(np.float32)
    assert np.array_equal(got, want)
    assert np.all((got >= -0.1) & (got < 0.1))

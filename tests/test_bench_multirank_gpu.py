"""GPU: bench.py's multi-rank path executed end to end.

The driver's scaling run launches ``bench.py`` under torchrun with one rank
per GPU over NCCL.  A gpurun box has one GPU, so here two ranks share it
(bench.py's ISINGLINK_BENCH_DEVICE hook) over gloo (two NCCL ranks may not
share a device); everything else -- the subcarrier shards, per-RE seeds keyed
by the global RE index, the Gray demapper, gather_to_rank0, the barrier and
max-over-ranks timing, the e2e host-buffer leg -- is the code the 8-GPU run
executes.  The gathered bits must equal the one-rank run's bit for bit
(harness/workers.py:17-38 partitioning).
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bench(tmp_path, world: int) -> tuple[dict, np.ndarray]:
    bits = tmp_path / f"bits_w{world}.npy"
    env = dict(os.environ, ISINGLINK_BENCH_BITS=str(bits), ISINGLINK_BENCH_DEVICE="0",
               ISINGLINK_BENCH_BACKEND="gloo")
    args = ["bench.py", "--gpus", str(world), "--steps", "2", "--warmup", "1",
            "--no-cpu-baseline", "--no-other-configs"]
    if world > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
               str(_port()), *args]
    else:
        cmd = [sys.executable, *args]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    return json.loads(lines[0]), np.load(bits)


def test_two_ranks_gather_the_one_rank_bits(tmp_path):
    one, b1 = _bench(tmp_path, 1)
    two, b2 = _bench(tmp_path, 2)
    assert b1.shape == (273 * 12 * 14, 16, 4) and b1.dtype == np.uint8  # 16-QAM: 2 x 2 bits
    assert np.array_equal(b1, b2)
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["config"]["parallelism"] == "subcarrier-shard x2"
    assert one["ser_check"] == pytest.approx(two["ser_check"], abs=0.02)  # rank 0's shard vs slot
    for line in (one, two):
        assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0

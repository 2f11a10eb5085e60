"""CPU, world_size 2 over gloo: the multi-GPU path's host logic.

Each rank detects its subcarrier shard of a (small) slot with per-RE seeds
keyed by the global RE index, then the decisions are gathered to rank 0 with
shard.gather_to_rank0 (the same code the NCCL path runs).  The gathered
result must equal the single-process result bit for bit.  The per-RE
detector here is the oracle (CPU); on the GPU the CUDA path plugs into the
same sharding/gather code (bench.py).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import isinglink_oracle as orc
from paper_2510_01579_b200.shard import gather_to_rank0, slot_shard

N_PRB = 1  # 12 subcarriers x 14 symbols = 168 REs
ORDER, NT = 4, 4


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _detect_range(lo, hi):
    levels, _ = orc.qam(ORDER)
    out = np.zeros((hi - lo, NT, 2), np.uint8)
    prm = orc.params(n_anneals=8, n_steps=32)
    for k, t in enumerate(range(lo, hi)):
        H, y, s2, _ = orc.uplink_instance(9, 12.0, 0, t, NT, NT, ORDER)
        r = orc.detect_cim(H, y, s2, ORDER, prm=prm, seed=orc.seed_of(9, 1, 0, t, 3))
        out[k] = np.stack([orc.level_index(r["x"].real, levels),
                           orc.level_index(r["x"].imag, levels)], -1)
    return out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shard = slot_shard(N_PRB, rank, world)
    local = torch.from_numpy(_detect_range(shard.re_start, shard.re_stop))
    got = gather_to_rank0(local, shard)
    if rank == 0:
        q.put(got.numpy())
    else:
        assert got is None
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_detection_gathers_identically():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = slot_shard(N_PRB, 0, 1).n_res
    assert got.shape == (n, NT, 2)
    assert np.array_equal(got, _detect_range(0, n))


def _gather_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shard = slot_shard(3, rank, world)  # 36 sc over 3 ranks -> 12, 12, 12 sc
    local = torch.arange(shard.re_start, shard.re_stop, dtype=torch.int64)[:, None].repeat(1, 2)
    got = gather_to_rank0(local.to(torch.uint8), shard)
    if rank == 0:
        q.put(got.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_is_slot_ordered(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = (np.arange(3 * 12 * 14)[:, None].repeat(2, 1)).astype(np.uint8)
    assert np.array_equal(got, want)

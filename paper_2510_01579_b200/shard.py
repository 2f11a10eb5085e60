"""Subcarrier sharding of a slot across GPUs (one process per GPU).

Resource elements of a slot are ordered subcarrier-major (``re = sc * 14 +
sym``) so a subcarrier range is a contiguous block of REs.  Ranks take
contiguous equal subcarrier blocks with the remainder on the last rank —
the reference's ``partition_blocks`` rule (harness/workers.py:17-25) applied
to subcarriers, the paper's split of the band across GPUs.
Every per-RE seed is keyed by the *global* RE index, so detections are
bit-identical for any number of GPUs.  Detection needs no exchange; the only
collective is the final gather of the detected (Gray-coded) bits to rank 0.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

SYMBOLS_PER_SLOT = 14
SUBCARRIERS_PER_PRB = 12


def partition_blocks(n_items: int, n_workers: int) -> list[tuple[int, int]]:
    """Contiguous [start, stop) blocks, remainder to the last block."""
    if n_workers < 1:
        raise ValueError("n_workers must be >= 1")
    n_workers = min(n_workers, max(n_items, 1))
    size = n_items // n_workers
    blocks = [(i * size, (i + 1) * size) for i in range(n_workers)]
    blocks[-1] = (blocks[-1][0], n_items)
    return blocks


@dataclass(frozen=True)
class SlotShard:
    n_prb: int
    rank: int
    world: int
    sc_start: int
    sc_stop: int

    @property
    def n_subcarriers(self) -> int:
        return self.n_prb * SUBCARRIERS_PER_PRB

    @property
    def n_res(self) -> int:
        return self.n_subcarriers * SYMBOLS_PER_SLOT

    @property
    def re_start(self) -> int:
        return self.sc_start * SYMBOLS_PER_SLOT

    @property
    def re_stop(self) -> int:
        return self.sc_stop * SYMBOLS_PER_SLOT

    @property
    def local_res(self) -> int:
        return self.re_stop - self.re_start


def slot_shard(n_prb: int, rank: int, world: int) -> SlotShard:
    n_sc = n_prb * SUBCARRIERS_PER_PRB
    blocks = partition_blocks(n_sc, world)
    if rank >= len(blocks):
        return SlotShard(n_prb, rank, world, n_sc, n_sc)
    a, b = blocks[rank]
    return SlotShard(n_prb, rank, world, a, b)


def gather_to_rank0(local: torch.Tensor, shard: SlotShard, group=None):
    """Gather per-rank [local_res, ...] tensors into the slot-ordered tensor
    on rank 0 (None elsewhere).  One NCCL all_gather of buffers padded to the
    largest shard, then trimmed and concatenated in rank order."""
    world = dist.get_world_size(group)
    if world == 1:
        return local
    blocks = partition_blocks(shard.n_subcarriers, world)
    sizes = [(b - a) * SYMBOLS_PER_SLOT for a, b in blocks] + [0] * (world - len(blocks))
    pad = max(sizes)
    buf = torch.zeros((pad,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    if dist.get_rank(group) != 0:
        return None
    return torch.cat([o[:s] for o, s in zip(out, sizes)], dim=0)

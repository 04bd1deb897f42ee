"""Batch sharding across the GPUs of one box.

Every sample is independent (no cross-sample op in the reference forward,
layers.hpp:99-211), so the batch is split into contiguous equal shards, one
per rank, with the weights replicated.  The forward has no collective; only
the logits come back to rank 0, gathered over NCCL (NVLink/NVSwitch) on GPU
or gloo in the CPU tests.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_rows(batch: int, rank: int, world: int):
    """[start, stop) rows of `rank`'s contiguous shard."""
    per = (batch + world - 1) // world
    start = min(batch, rank * per)
    return start, min(batch, start + per)


def gather_logits(local: torch.Tensor, batch: int, group=None) -> torch.Tensor:
    """All-gather the per-rank logit shards; returns the full [batch, n] tensor
    (meaningful on every rank; rank 0 is the consumer).  Shards are padded to
    equal length for the collective and trimmed afterwards."""
    world = dist.get_world_size(group)
    per = (batch + world - 1) // world
    n = local.shape[1]
    padded = torch.zeros((per, n), dtype=local.dtype, device=local.device)
    padded[: local.shape[0]] = local
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    rows = []
    for r in range(world):
        s, e = shard_rows(batch, r, world)
        rows.append(parts[r][: e - s])
    return torch.cat(rows, 0)

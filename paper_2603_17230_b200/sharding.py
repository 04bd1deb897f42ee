"""Batch sharding across the GPUs of one box.

Every sample is independent (no cross-sample op in the reference forward,
layers.hpp:99-211), so the global batch is split into contiguous equal shards,
one per rank (kan_shard_rows), with the weights replicated.  The forward has
no collective; only the logits come back to rank 0, gathered over NCCL
(NVLink/NVSwitch) on GPUs, or gloo in the CPU tests.  This replaces the
reference's serial chunk loop of predict (eval.hpp:255-276) at box scale.

In-process multi-device use goes through kan_engine_forward_sharded
(engine.forward_sharded); the torchrun path (one process per GPU, as bench.py
runs) uses LogitGather below.
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist


def shard_rows(batch: int, rank: int, world: int):
    """[start, stop) rows of `rank`'s contiguous shard (ceil(batch/world) each;
    the same rule as kan_shard_rows in the C ABI)."""
    per = (batch + world - 1) // world
    start = min(batch, rank * per)
    return start, min(batch, start + per)


class LogitGather:
    """Gather of per-rank logit shards to rank 0 with preallocated buffers (no
    allocation per step).  Shards are padded to ceil(batch/world) rows for the
    collective and trimmed on rank 0."""

    def __init__(self, batch: int, n_out: int, dtype, device, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.batch = batch
        self.per = (batch + self.world - 1) // self.world
        self.rows = shard_rows(batch, self.rank, self.world)
        self.send = torch.zeros((self.per, n_out), dtype=dtype, device=device)
        self.recv = (torch.empty((self.world * self.per, n_out), dtype=dtype, device=device)
                     if self.rank == 0 else None)
        self.parts = list(self.recv.view(self.world, self.per, n_out).unbind(0)) if self.rank == 0 else None

    def __call__(self, local: torch.Tensor) -> Optional[torch.Tensor]:
        """Gather this rank's [rows, n_out] logits; returns the full
        [batch, n_out] logits on rank 0 (a view of the receive buffer), None
        elsewhere."""
        n = local.shape[0]
        assert n == self.rows[1] - self.rows[0], "shard size mismatch"
        self.send[:n].copy_(local)
        dist.gather(self.send, self.parts, dst=0, group=self.group)
        if self.rank != 0:
            return None
        if self.batch == self.world * self.per:
            return self.recv
        spans = [shard_rows(self.batch, r, self.world) for r in range(self.world)]
        return torch.cat([self.parts[r][: b - a] for r, (a, b) in enumerate(spans)], 0)


def sharded_forward(forward: Callable[[torch.Tensor], torch.Tensor], x_global: torch.Tensor, n_out: int,
                    group=None) -> Optional[torch.Tensor]:
    """The torchrun data path in one call: this rank's contiguous shard of
    x_global -> forward(shard) -> logits gathered to rank 0 (returned there)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    s, e = shard_rows(x_global.shape[0], rank, world)
    y = forward(x_global[s:e])
    g = LogitGather(x_global.shape[0], n_out, y.dtype, y.device, group)
    return g(y)

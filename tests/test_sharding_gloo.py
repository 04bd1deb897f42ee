"""Multi-process (world_size 2, gloo, CPU) test of the batch-sharding path:
contiguous shards, per-rank forward of independent samples, logits gathered
back in order -- the host-side logic bench.py runs over NCCL on GPUs."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_17230_b200.sharding import gather_logits, shard_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, batch, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    full = torch.from_numpy(rng.standard_normal((batch, 10)).astype(np.float32))
    s, e = shard_rows(batch, rank, world)
    local = full[s:e] * 1.0  # stand-in for the per-rank forward of its own rows
    out = gather_logits(local, batch)
    if rank == 0:
        q.put(bool(torch.equal(out, full)))
    dist.destroy_process_group()


def test_shard_rows_partition():
    for batch in (0, 1, 7, 4096, 8193):
        for world in (1, 2, 3, 8):
            spans = [shard_rows(batch, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b


def test_gather_logits_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    for batch in (4096, 8193):
        procs = [ctx.Process(target=_worker, args=(r, 2, port, batch, q)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0
        assert q.get(timeout=10)
        port = _free_port()

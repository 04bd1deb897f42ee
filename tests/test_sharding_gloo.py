"""Multi-process (world_size 2, gloo, CPU) test of the batch-sharding data path
bench.py runs over NCCL on GPUs: contiguous shards (kan_shard_rows' rule), a
real per-rank forward of the rank's own rows, and the logits gathered to rank 0
in order (sharding.LogitGather / sharded_forward).  On CPU the per-rank forward
is the oracle's integer LUT forward of a reduced ResKAN18 (the engine needs a
GPU); the gathered logits must equal the oracle's full-batch forward exactly."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_17230_b200 import configs
from paper_2603_17230_b200.sharding import LogitGather, shard_rows, sharded_forward

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _model():
    layers = configs.reskan18_layers(width=(8, 16), n_classes=10, in_ch=3)
    desc = {"name": "reskan-tiny", "grid": {"intervals": 5, "degree": 3}, "input": [3, 8, 8],
            "conv_output": "floor", "layers": layers}
    wl = configs.Workload("t", "t", [0], 5, 3, 1, 0.05, silu=False, wscheme=0, lut_h=3,
                          input_shape=desc["input"], layers=layers, extra={"descriptor": {"conv_output": "floor"}})
    return desc, wl


def _worker(rank, world, port, batch, q):
    import sys
    sys.path.insert(0, ROOT)
    from oracle.pyoracle import Oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    desc, wl = _model()
    Ws, Bs = wl.weights()
    x = torch.from_numpy(wl.inputs(batch, seed=3))

    def forward(rows):  # this rank's forward of its own rows only
        y = o.int_model_forward(desc, Ws, Bs, rows.numpy(), 8, 3, 0, 8)
        return torch.from_numpy(y.astype(np.float32))
    out = sharded_forward(forward, x, 10)
    # a second step through the same preallocated gather
    s, e = shard_rows(batch, rank, world)
    g = LogitGather(batch, 10, torch.float32, torch.device("cpu"))
    out2 = g(forward(x[s:e]))
    if rank == 0:
        full = forward(x)
        q.put(bool(torch.equal(out, full)) and bool(torch.equal(out2, full)))
    else:
        q.put(out is None and out2 is None)
    dist.destroy_process_group()


def test_shard_rows_partition():
    from paper_2603_17230_b200.engine import shard_rows as abi_shard_rows
    for batch in (0, 1, 7, 4096, 8193):
        for world in (1, 2, 3, 8):
            spans = [shard_rows(batch, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
            assert spans == [abi_shard_rows(batch, r, world) for r in range(world)]  # same rule as the C ABI


def test_sharded_forward_world2_gloo():
    ctx = mp.get_context("spawn")
    for batch in (6, 7):  # even and ragged shards
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, 2, port, batch, q)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(300)
            assert p.exitcode == 0
        assert q.get(timeout=10) and q.get(timeout=10)

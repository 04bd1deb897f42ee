"""GPU tests of the multi-engine forward behind the C ABI
(kan_engine_forward_sharded / _host): contiguous shards,
one engine per shard, logits landing in one buffer on engines[0]'s device.
This box has one GPU, so the shards are engines sharing it; the logits must be
bit-identical to one engine's forward of the whole batch (integer LUT path:
rows are independent and each row's arithmetic is fixed).  Also: the engine
option API, the launch plan probe and configure's int32 headroom check."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2603_17230_b200 import Engine, EvalOptions, configs, engine  # noqa: E402


def reskan_small():
    layers = configs.reskan18_layers(width=(16, 32), n_classes=10, in_ch=3)
    return configs.Workload("rs", "rs", [0], 5, 3, 1, 0.05, silu=False, wscheme=0, lut_h=3,
                            input_shape=[3, 16, 16], layers=layers,
                            extra={"descriptor": {"conv_output": "floor"}})


def make(wl, n, **opt):
    Ws, Bs = wl.weights()
    out = []
    for _ in range(n):
        e = Engine(wl.descriptor(), 0)
        for i, (w, b) in enumerate(zip(Ws, Bs)):
            e.set_coeffs(i, w, b)
        e.configure(EvalOptions(**wl.eval_options(), **opt))
        out.append(e)
    return out


@pytest.mark.parametrize("n,batch", [(2, 64), (3, 50), (4, 3), (2, 1)])
def test_forward_sharded_equals_single_engine(n, batch):
    wl = reskan_small()
    engs = make(wl, n + 1)
    x = wl.inputs(batch, seed=n)
    xd = torch.from_numpy(x).cuda()
    ref = engs[0].model_forward(xd).cpu().numpy()
    group = engs[1:]
    shards = []
    for g in range(n):
        a, b = engine.shard_rows(batch, g, n)
        shards.append(xd[a:b].contiguous() if b > a else None)
    out = torch.full((batch, wl.out_size), float("nan"), device="cuda")
    streams = [torch.cuda.Stream() for _ in range(n)]
    engine.forward_sharded(group, shards, out, streams=streams)
    torch.cuda.current_stream().wait_stream(streams[0])
    np.testing.assert_array_equal(out.cpu().numpy(), ref)
    # misaligned destination offsets take the staging copy
    out2 = torch.full((batch + 1, wl.out_size), float("nan"), device="cuda")
    engine.forward_sharded(group, shards, out2[1:])
    np.testing.assert_array_equal(out2[1:].cpu().numpy(), ref)
    # host buffers: H2D, forward and D2H on each engine's own stream
    np.testing.assert_array_equal(engine.forward_sharded_host(group, x), ref)


def test_forward_sharded_rejects_mismatched_engines():
    wl = reskan_small()
    a, = make(wl, 1)
    b, = make(wl, 1, split_k=1)
    mlp = configs.get("c1")
    c, = make(mlp, 1)
    x = torch.zeros((4, wl.input_size), device="cuda")
    out = torch.empty((4, 10), device="cuda")
    with pytest.raises(ValueError):
        engine.forward_sharded([a, c], [x[:2], x[2:]], out)
    with pytest.raises(ValueError):
        engine.forward_sharded([a, a], [x[:2], x[2:]], out)
    engine.forward_sharded([a, b], [x[:2], x[2:]], out)  # same model, other tiling: fine


def test_options_and_launch_plan():
    wl = reskan_small()
    e, = make(wl, 1)
    with pytest.raises(ValueError):
        e.set_option("tables", 7)
    e.set_option("record_plan", 1)
    x = torch.from_numpy(wl.inputs(4, seed=1)).cuda()
    e.model_forward(x)
    plan = e.last_plan.strip().splitlines()
    assert len(plan) == e.last_launches
    assert plan[0].startswith("im2col_levels") or plan[0].startswith("nchw_to_nhwc")
    assert sum(p.startswith(("gather", "conv3", "convw", "small_layer")) for p in plan) == wl.n_kan
    e.set_option("record_plan", 0)
    e.model_forward(x)
    assert e.last_plan == ""


def test_int32_headroom_is_checked_at_configure():
    """A layer whose worst-case int32 accumulator could overflow is refused
    (SURVEY 7.2): 40,000 inputs x (255 + 2) x 127 exceeds 2^31 - 1."""
    n_in = 40000
    desc = {"name": "wide", "grid": {"intervals": 5, "degree": 3}, "input": [n_in],
            "layers": [{"type": "linear", "n_in": n_in, "n_out": 1}]}
    e = Engine(desc, 0)
    e.set_coeffs(0, np.full((n_in * 8, 1), 0.1), np.full((n_in, 1), 0.1))
    with pytest.raises(NotImplementedError, match="int32 accumulator"):
        e.configure(EvalOptions(mode="bspline-lut", lut_k=8, lut_h=8, bits_w=8, w_scheme=1, silu_base=True))
    # the same width at h = 3 fits: 40,000 x ((7 + 2) x 127 + 255 x 127) < 2^31
    e.configure(EvalOptions(mode="bspline-lut", lut_k=8, lut_h=3, bits_w=8, w_scheme=1, silu_base=True))

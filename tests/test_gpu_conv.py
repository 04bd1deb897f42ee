"""GPU parity of the conv path (implicit im2col through 4D TMA) and of the
ResKAN18 building blocks (stride-2 convs, 1x1 projection shortcuts, residual
adds, pooling, flatten), through the C ABI, against the CPU oracle
(oracle/pyoracle.py Oracle.int_model_forward) and the compiled reference.

Bar: bit-exact on the integer LUT path; 1e-2 norm-relative on the bf16 path.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2603_17230_b200 import (  # noqa: E402
    Engine, EvalOptions, W_PER_CHANNEL_SYM, W_PER_TENSOR_ASYM, configs)


def conv_desc(C, H, W, co, k, s, p, floor=False):
    d = {"name": "conv", "grid": {"intervals": 5, "degree": 3}, "input": [C, H, W],
         "layers": [{"type": "conv", "c_in": C, "c_out": co, "kernel": k, "stride": s,
                     "padding": p}]}
    if floor:
        d["conv_output"] = "floor"
    return d


def weights_for(desc, G=5, P=3, seed=0, std=0.05, silu=True):
    wl = configs.Workload("t", "t", [0], G, P, 1, std, silu=silu, seed=seed,
                          input_shape=desc["input"], layers=desc["layers"])
    return wl.weights()


def build(desc, Ws, Bs, engine_options=None, **opts):
    e = Engine(desc, 0)
    for i, (w, b) in enumerate(zip(Ws, Bs)):
        e.set_coeffs(i, w, b)
    for k, v in (engine_options or {}).items():
        e.set_option(k, v)
    e.configure(EvalOptions(**opts))
    return e


def to_dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


CONV_CASES = [
    # C, H, W, c_out, k, s, p, silu, wscheme, batch, split
    (64, 32, 32, 64, 3, 1, 1, True, W_PER_CHANNEL_SYM, 2, 0),   # C4 shape
    (16, 8, 8, 24, 3, 1, 1, False, W_PER_CHANNEL_SYM, 5, 0),    # 2 images per M tile, ragged
    (3, 16, 16, 16, 3, 1, 1, True, W_PER_CHANNEL_SYM, 3, 0),    # stem: c_in < one chunk
    (8, 8, 8, 8, 3, 1, 1, False, W_PER_TENSOR_ASYM, 4, 0),      # reference weight scheme
    (64, 16, 16, 32, 3, 1, 1, True, W_PER_CHANNEL_SYM, 2, 2),   # split-K over a cluster
    (32, 4, 4, 300, 3, 1, 1, True, W_PER_CHANNEL_SYM, 9, 0),    # 8 images per tile, 2 N tiles
    (5, 8, 8, 7, 1, 1, 0, True, W_PER_CHANNEL_SYM, 4, 0),       # 1x1
    (2, 9, 11, 20, 5, 2, 2, True, W_PER_CHANNEL_SYM, 3, 0),     # 5x5 s2 stem (explicit im2col)
]


@pytest.mark.parametrize("C,H,W,co,k,s,p,silu,ws,batch,split", CONV_CASES)
def test_conv_layer_bit_exact(oracle, C, H, W, co, k, s, p, silu, ws, batch, split):
    desc = conv_desc(C, H, W, co, k, s, p)
    Ws, Bs = weights_for(desc, seed=C + co, silu=silu)
    x = np.random.default_rng(C * 7 + co).uniform(-1.05, 1.05, (batch, C * H * W)).astype(np.float32)
    e = build(desc, Ws, Bs, mode="bspline-lut", lut_k=8, lut_h=8, bits_w=8, w_scheme=ws,
              silu_base=silu, split_k=split)
    y = e.model_forward(to_dev(x)).cpu().numpy()
    yo = oracle.int_model_forward(desc, Ws, Bs, x, 8, 8, ws, 8)
    np.testing.assert_array_equal(y, yo.astype(np.float32).reshape(batch, -1))


def test_conv_reference_scheme_matches_reference_conv(oracle, ref):
    """Reference weight scheme (per-tensor u8, no SiLU): the GPU conv equals
    convkan_forward with LutBasis (layers.hpp:162-190) to fp32 rounding."""
    desc = conv_desc(8, 8, 8, 6, 3, 1, 1)
    Ws, _ = weights_for(desc, seed=3, silu=False)
    x = np.random.default_rng(3).uniform(-1, 1, (3, 8 * 64)).astype(np.float32)
    e = build(desc, Ws, [None], mode="bspline-lut", lut_k=8, lut_h=8, bits_w=8,
              w_scheme=W_PER_TENSOR_ASYM)
    y = e.model_forward(to_dev(x)).cpu().numpy().reshape(3, 6, 8, 8)
    for n in range(3):
        r = ref.conv_forward(5, 3, x[n].reshape(8, 8, 8).astype(np.float64), Ws[0], 6, 3, 1, 1,
                             mode=1, k=8, h=8, bits_w=8)
        assert rel_err(y[n], r) < 1e-6


@pytest.mark.parametrize("k,s,p", [(3, 2, 1), (1, 2, 0)])
def test_strided_conv_on_levels_bit_exact(oracle, k, s, p):
    """Stride-2 convs read stored NHWC levels through TMA element strides."""
    desc = {"name": "s2", "grid": {"intervals": 5, "degree": 3}, "input": [3, 16, 16],
            "conv_output": "floor",
            "layers": [{"type": "conv", "c_in": 3, "c_out": 32, "kernel": 3, "stride": 1, "padding": 1},
                       {"type": "conv", "c_in": 32, "c_out": 40, "kernel": k, "stride": s, "padding": p}]}
    Ws, Bs = weights_for(desc, seed=k)
    x = np.random.default_rng(k).uniform(-1, 1, (3, 3 * 256)).astype(np.float32)
    e = build(desc, Ws, Bs, mode="bspline-lut", lut_k=8, lut_h=8, bits_w=8,
              w_scheme=W_PER_CHANNEL_SYM, silu_base=True)
    y = e.model_forward(to_dev(x)).cpu().numpy()
    yo = oracle.int_model_forward(desc, Ws, Bs, x, 8, 8, W_PER_CHANNEL_SYM, 8)
    np.testing.assert_array_equal(y, yo.astype(np.float32).reshape(3, -1))


@pytest.mark.parametrize("h", [3, 8])
@pytest.mark.parametrize("split", [0, 1])
def test_small_reskan_bit_exact(oracle, h, split):
    """ResKAN18 topology at reduced width / resolution: stem, identity and
    projection residual blocks, stride 2, global average pool, linear head.
    split_k=1 keeps every launch persistent, so the straight-line epilogue
    instantiations (levels, residual + levels, fp32 + residual + sidecar) run."""
    layers = configs.reskan18_layers(width=(16, 32), n_classes=10, in_ch=3)
    desc = {"name": "reskan-small", "grid": {"intervals": 5, "degree": 3}, "input": [3, 16, 16],
            "conv_output": "floor", "layers": layers}
    Ws, Bs = weights_for(desc, seed=h)
    x = np.random.default_rng(h).uniform(-1, 1, (6, 3 * 256)).astype(np.float32)
    e = build(desc, Ws, Bs, mode="bspline-lut", lut_k=8, lut_h=h, bits_w=8,
              w_scheme=W_PER_CHANNEL_SYM, silu_base=True, split_k=split)
    y = e.model_forward(to_dev(x)).cpu().numpy()
    yo = oracle.int_model_forward(desc, Ws, Bs, x, 8, h, W_PER_CHANNEL_SYM, 8)
    np.testing.assert_array_equal(y, yo.astype(np.float32))
    # one launch per KAN layer + the input transpose + the pooling kernel
    assert e.last_launches == len(Ws) + 2


def test_maxpool_flatten_linear_bit_exact(oracle):
    """conv -> maxpool -> flatten -> linear (the reference's LeKAN-style stack):
    the linear layer's rows are permuted to the stored NHWC order."""
    desc = {"name": "cnn", "grid": {"intervals": 5, "degree": 3}, "input": [1, 16, 16],
            "layers": [{"type": "conv", "c_in": 1, "c_out": 8, "kernel": 3, "stride": 1, "padding": 1},
                       {"type": "maxpool", "window": 2},
                       {"type": "flatten"},
                       {"type": "linear", "n_in": 8 * 8 * 8, "n_out": 10}]}
    Ws, Bs = weights_for(desc, seed=5)
    x = np.random.default_rng(5).uniform(-1, 1, (7, 256)).astype(np.float32)
    e = build(desc, Ws, Bs, mode="bspline-lut", lut_k=8, lut_h=8, bits_w=8,
              w_scheme=W_PER_CHANNEL_SYM, silu_base=True)
    y = e.model_forward(to_dev(x)).cpu().numpy()
    yo = oracle.int_model_forward(desc, Ws, Bs, x, 8, 8, W_PER_CHANNEL_SYM, 8)
    np.testing.assert_array_equal(y, yo.astype(np.float32))


def test_bf16_conv_vs_reference(ref):
    """bf16 path (fp32 Cox-de Boor basis -> bf16 tcgen05): 1e-2 norm-relative
    against the reference's fp64 convkan_forward."""
    desc = conv_desc(16, 8, 8, 16, 3, 1, 1)
    Ws, _ = weights_for(desc, seed=11, silu=False)
    x = np.random.default_rng(11).uniform(-1, 1, (2, 16 * 64)).astype(np.float32)
    e = build(desc, Ws, [None], mode="bf16")
    y = e.model_forward(to_dev(x)).cpu().numpy().reshape(2, 16, 8, 8)
    r = np.stack([ref.conv_forward(5, 3, x[n].reshape(16, 8, 8).astype(np.float64), Ws[0], 16, 3,
                                   1, 1) for n in range(2)])
    assert rel_err(y, r) < 1e-2


# ky-shared 3x3 kernel (kan_conv3.cuh): taken for 3x3/s1/p1 convs whose tile
# grid fills the GPU (>= 148 tiles); smaller grids use the general kernel.
CONV3_CASES = [
    # C, H, W, c_out, silu, batch
    (64, 32, 32, 64, True, 20),    # C4 shape, 160 tiles
    (40, 16, 16, 48, False, 80),   # partial channel chunk, 16x16 maps
    (32, 32, 32, 24, True, 19),    # one chunk
    (32, 20, 32, 40, True, 31),    # 155 tiles: odd, the last weight-multicast pair has one tile
]


@pytest.mark.parametrize("C,H,W,co,silu,batch", CONV3_CASES)
def test_conv3_kernel_bit_exact(oracle, C, H, W, co, silu, batch):
    desc = conv_desc(C, H, W, co, 3, 1, 1)
    Ws, Bs = weights_for(desc, seed=C + batch, silu=silu)
    x = np.random.default_rng(C + co).uniform(-1.05, 1.05, (batch, C * H * W)).astype(np.float32)
    e = build(desc, Ws, Bs, mode="bspline-lut", lut_k=8, lut_h=8, bits_w=8, w_scheme=W_PER_CHANNEL_SYM,
              silu_base=silu)
    y = e.model_forward(to_dev(x)).cpu().numpy()
    yo = oracle.int_model_forward(desc, Ws, Bs, x, 8, 8, W_PER_CHANNEL_SYM, 8)
    np.testing.assert_array_equal(y, yo.astype(np.float32).reshape(batch, -1))


def test_conv3_matches_general_kernel_in_a_residual_stage():
    """Stage-1 blocks at 32x32 take the ky-shared kernel (fp32-stored block
    inputs and level inputs); the result is bit-identical to the general
    gather-GEMM kernel (option no_conv3)."""
    layers = configs.reskan18_layers(width=(16, 32), n_classes=10, in_ch=3)
    desc = {"name": "r", "grid": {"intervals": 5, "degree": 3}, "input": [3, 32, 32],
            "conv_output": "floor", "layers": layers}
    Ws, Bs = weights_for(desc, seed=21)
    x = np.random.default_rng(21).uniform(-1, 1, (20, 3 * 1024)).astype(np.float32)
    opts = dict(mode="bspline-lut", lut_k=8, lut_h=3, bits_w=8, w_scheme=W_PER_CHANNEL_SYM, silu_base=True)
    y3 = build(desc, Ws, Bs, **opts).model_forward(to_dev(x)).cpu().numpy()
    yg = build(desc, Ws, Bs, engine_options={"no_conv3": 1}, **opts).model_forward(to_dev(x)).cpu().numpy()
    np.testing.assert_array_equal(y3, yg)


@pytest.mark.parametrize("k,s,p", [(3, 1, 1), (3, 2, 1), (1, 1, 0)])
def test_stem_im2col_matches_implicit_conv(k, s, p):
    """Stem convs (model input, c_in < 16) run as a dense GEMM over an explicit
    level im2col; the result is bit-identical to the implicit-im2col conv
    kernel over the transposed input (option no_im2col)."""
    desc = conv_desc(3, 16, 16, 32, k, s, p, floor=True)
    desc["layers"].append({"type": "conv", "c_in": 32, "c_out": 8, "kernel": 1, "stride": 1, "padding": 0})
    Ws, Bs = weights_for(desc, seed=k + s)
    x = np.random.default_rng(k * s).uniform(-1.05, 1.05, (5, 3 * 256)).astype(np.float32)
    opts = dict(mode="bspline-lut", lut_k=8, lut_h=8, bits_w=8, w_scheme=W_PER_CHANNEL_SYM, silu_base=True)
    yi = build(desc, Ws, Bs, **opts).model_forward(to_dev(x)).cpu().numpy()
    yc = build(desc, Ws, Bs, engine_options={"no_im2col": 1}, **opts).model_forward(to_dev(x)).cpu().numpy()
    np.testing.assert_array_equal(yi, yc)


# window-shared 3x3 kernel (kan_convw.cuh): 8 images per tile, all nine taps
# from one expanded window; taken for 3x3/s1/p1 convs on stored levels with
# 16- or 32-wide maps and no SiLU term.  Inputs are stored levels, so the
# layer under test follows a 1x1 conv (which writes the levels).
CONVW_CASES = [
    # C, H, W, c_out, wscheme, batch
    (64, 32, 32, 64, W_PER_TENSOR_ASYM, 16),   # C5 stage 1, the reference scheme
    (64, 32, 32, 64, W_PER_CHANNEL_SYM, 13),   # partial image group
    (128, 16, 16, 128, W_PER_TENSOR_ASYM, 9),  # C5 stage 2
    (32, 16, 16, 256, W_PER_CHANNEL_SYM, 8),   # BN 256, one output row per tile
    (16, 16, 16, 40, W_PER_TENSOR_ASYM, 11),   # ragged 16-column group
    (8, 16, 16, 300, W_PER_CHANNEL_SYM, 3),    # two N tiles, the second ragged
    (32, 8, 8, 256, W_PER_TENSOR_ASYM, 20),    # 8-wide maps: 16 images per tile, partial group
    (64, 4, 4, 512, W_PER_CHANNEL_SYM, 40),    # 4-wide maps: 32 images per tile, two N tiles
    (16, 8, 8, 24, W_PER_TENSOR_ASYM, 5),      # 8-wide, one partial group, ragged N
]


@pytest.mark.parametrize("C,H,W,co,ws,batch", CONVW_CASES)
def test_convw_kernel_bit_exact(oracle, C, H, W, co, ws, batch):
    desc = conv_desc(C, H, W, C, 1, 1, 0)
    desc["layers"].append({"type": "conv", "c_in": C, "c_out": co, "kernel": 3, "stride": 1, "padding": 1})
    # a 1x1 consumer, so the layer under test writes a stored (NHWC) tensor
    desc["layers"].append({"type": "conv", "c_in": co, "c_out": 8, "kernel": 1, "stride": 1, "padding": 0})
    Ws, Bs = weights_for(desc, seed=C + co, silu=False)
    x = np.random.default_rng(C * co).uniform(-1.05, 1.05, (batch, C * H * W)).astype(np.float32)
    opts = dict(mode="bspline-lut", lut_k=8, lut_h=3, bits_w=8, w_scheme=ws, silu_base=False)
    e = build(desc, Ws, Bs, **opts)
    e.set_option("record_plan", 1)
    y = e.model_forward(to_dev(x)).cpu().numpy()
    assert "convw layer=1" in e.last_plan
    yg = build(desc, Ws, Bs, engine_options={"no_convw": 1, "no_conv3": 1}, **opts).model_forward(to_dev(x)).cpu().numpy()
    np.testing.assert_array_equal(y, yg)
    yo = oracle.int_model_forward(desc, Ws, Bs, x, 8, 3, ws, 8)
    np.testing.assert_array_equal(y, yo.astype(np.float32).reshape(batch, -1))


@pytest.mark.parametrize("ws", [W_PER_TENSOR_ASYM, W_PER_CHANNEL_SYM])
def test_convw_in_residual_stages_bit_exact(oracle, ws):
    """Reduced-width ResKAN18 (all four stages: 32/16/8/4-wide maps) at
    32x32 without the SiLU term: the stride-1 convs take kan_convw (levels
    out; fp32 + residual + levels sidecar out; residual then levels), batch 21
    (partial image groups of 8, 16 and 32)."""
    layers = configs.reskan18_layers(width=(8, 16, 32, 64), n_classes=10, in_ch=3)
    desc = {"name": "r", "grid": {"intervals": 5, "degree": 3}, "input": [3, 32, 32],
            "conv_output": "floor", "layers": layers}
    Ws, Bs = weights_for(desc, seed=23, silu=False)
    x = np.random.default_rng(23).uniform(-1, 1, (21, 3 * 1024)).astype(np.float32)
    opts = dict(mode="bspline-lut", lut_k=8, lut_h=3, bits_w=8, w_scheme=ws, silu_base=False)
    e = build(desc, Ws, Bs, **opts)
    e.set_option("record_plan", 1)
    y = e.model_forward(to_dev(x)).cpu().numpy()
    assert e.last_plan.count("convw") >= 12
    yg = build(desc, Ws, Bs, engine_options={"no_convw": 1}, **opts).model_forward(to_dev(x)).cpu().numpy()
    np.testing.assert_array_equal(y, yg)
    yo = oracle.int_model_forward(desc, Ws, Bs, x, 8, 3, ws, 8)
    np.testing.assert_array_equal(y, yo.astype(np.float32))


@pytest.mark.parametrize("C,H,co,ws,batch", [
    (16, 32, 32, W_PER_TENSOR_ASYM, 11),   # 32x32 -> 16x16, partial image group
    (64, 32, 128, W_PER_CHANNEL_SYM, 8),   # the ResKAN18 stage-2 entry conv
    (8, 64, 24, W_PER_TENSOR_ASYM, 3),     # 64x64 -> 32x32: two 16-column blocks, ragged N
])
def test_convw_stride2_bit_exact(oracle, C, H, co, ws, batch):
    """Stride-2 3x3 pad-1 convs onto 16-wide multiples take kan_convw's
    stride-2 form (every other window pixel, a 512-byte core-matrix stride)."""
    desc = conv_desc(C, H, H, C, 1, 1, 0, floor=True)
    desc["layers"].append({"type": "conv", "c_in": C, "c_out": co, "kernel": 3, "stride": 2, "padding": 1})
    desc["layers"].append({"type": "conv", "c_in": co, "c_out": 8, "kernel": 1, "stride": 1, "padding": 0})
    Ws, Bs = weights_for(desc, seed=C + co + 1, silu=False)
    x = np.random.default_rng(C * co + 1).uniform(-1.05, 1.05, (batch, C * H * H)).astype(np.float32)
    opts = dict(mode="bspline-lut", lut_k=8, lut_h=3, bits_w=8, w_scheme=ws, silu_base=False)
    e = build(desc, Ws, Bs, **opts)
    e.set_option("record_plan", 1)
    y = e.model_forward(to_dev(x)).cpu().numpy()
    assert "convw layer=1" in e.last_plan
    yg = build(desc, Ws, Bs, engine_options={"no_convw": 1}, **opts).model_forward(to_dev(x)).cpu().numpy()
    np.testing.assert_array_equal(y, yg)
    yo = oracle.int_model_forward(desc, Ws, Bs, x, 8, 3, ws, 8)
    np.testing.assert_array_equal(y, yo.astype(np.float32).reshape(batch, -1))


# kan_convw with the SiLU base term (per-channel weights): one extra 32-byte
# K block of SiLU codes per 32 channels, against the base weights.
CONVW_SILU_CASES = [
    # C, H, W, c_out, batch
    (64, 32, 32, 64, 13),    # C5pc stage 1, partial image group
    (32, 16, 16, 128, 9),    # one 32-channel group, 16-wide maps
    (64, 8, 8, 256, 20),     # 8-wide maps, two N tiles
    (32, 4, 4, 40, 40),      # 4-wide maps, ragged N
]


@pytest.mark.parametrize("C,H,W,co,batch", CONVW_SILU_CASES)
def test_convw_silu_bit_exact(oracle, C, H, W, co, batch):
    desc = conv_desc(C, H, W, C, 1, 1, 0)
    desc["layers"].append({"type": "conv", "c_in": C, "c_out": co, "kernel": 3, "stride": 1, "padding": 1})
    desc["layers"].append({"type": "conv", "c_in": co, "c_out": 8, "kernel": 1, "stride": 1, "padding": 0})
    Ws, Bs = weights_for(desc, seed=C + co + 2, silu=True)
    x = np.random.default_rng(C * co + 2).uniform(-1.05, 1.05, (batch, C * H * W)).astype(np.float32)
    opts = dict(mode="bspline-lut", lut_k=8, lut_h=8, bits_w=8, w_scheme=W_PER_CHANNEL_SYM, silu_base=True)
    e = build(desc, Ws, Bs, **opts)
    e.set_option("record_plan", 1)
    y = e.model_forward(to_dev(x)).cpu().numpy()
    assert "convw layer=1" in e.last_plan
    yg = build(desc, Ws, Bs, engine_options={"no_convw": 1, "no_conv3": 1}, **opts).model_forward(to_dev(x)).cpu().numpy()
    np.testing.assert_array_equal(y, yg)
    yo = oracle.int_model_forward(desc, Ws, Bs, x, 8, 8, W_PER_CHANNEL_SYM, 8)
    np.testing.assert_array_equal(y, yo.astype(np.float32).reshape(batch, -1))


@pytest.mark.parametrize("C,H,W,co,silu,ws,batch", [
    (64, 32, 32, 64, True, W_PER_CHANNEL_SYM, 11),    # the C4 layer: NCHW model input and output
    (32, 16, 16, 40, True, W_PER_CHANNEL_SYM, 20),    # ragged N
    (64, 32, 32, 64, False, W_PER_TENSOR_ASYM, 9),    # the reference scheme
    (16, 8, 8, 300, False, W_PER_CHANNEL_SYM, 21),    # 8-wide maps, two N tiles
])
def test_convw_model_output_nchw_bit_exact(oracle, C, H, W, co, silu, ws, batch):
    """A single 3x3 conv as the whole model (C4): the NCHW input is transposed
    to NHWC levels, kan_convw writes the fp32 NCHW model output."""
    desc = conv_desc(C, H, W, co, 3, 1, 1)
    Ws, Bs = weights_for(desc, seed=C + co + 3, silu=silu)
    x = np.random.default_rng(C * co + 3).uniform(-1.05, 1.05, (batch, C * H * W)).astype(np.float32)
    opts = dict(mode="bspline-lut", lut_k=8, lut_h=8, bits_w=8, w_scheme=ws, silu_base=silu)
    e = build(desc, Ws, Bs, **opts)
    e.set_option("record_plan", 1)
    y = e.model_forward(to_dev(x)).cpu().numpy()
    assert "convw layer=0" in e.last_plan
    yg = build(desc, Ws, Bs, engine_options={"no_convw": 1, "no_conv3": 1}, **opts).model_forward(to_dev(x)).cpu().numpy()
    np.testing.assert_array_equal(y, yg)
    yo = oracle.int_model_forward(desc, Ws, Bs, x, 8, 8, ws, 8)
    np.testing.assert_array_equal(y, yo.astype(np.float32).reshape(batch, -1))


def test_convw_silu_in_residual_stages_bit_exact(oracle):
    """Reduced-width ResKAN18 (32/64 channels) with per-channel weights and the
    SiLU term: the stride-1 convs take kan_convw's SiLU form (levels out; fp32
    + residual + sidecar out), bit-identical to the general kernel and the oracle."""
    layers = configs.reskan18_layers(width=(32, 64), n_classes=10, in_ch=3)
    desc = {"name": "r", "grid": {"intervals": 5, "degree": 3}, "input": [3, 32, 32],
            "conv_output": "floor", "layers": layers}
    Ws, Bs = weights_for(desc, seed=29, silu=True)
    x = np.random.default_rng(29).uniform(-1, 1, (11, 3 * 1024)).astype(np.float32)
    opts = dict(mode="bspline-lut", lut_k=8, lut_h=3, bits_w=8, w_scheme=W_PER_CHANNEL_SYM, silu_base=True)
    e = build(desc, Ws, Bs, **opts)
    e.set_option("record_plan", 1)
    y = e.model_forward(to_dev(x)).cpu().numpy()
    assert e.last_plan.count("convw") >= 6
    yg = build(desc, Ws, Bs, engine_options={"no_convw": 1, "no_conv3": 1}, **opts).model_forward(to_dev(x)).cpu().numpy()
    np.testing.assert_array_equal(y, yg)
    yo = oracle.int_model_forward(desc, Ws, Bs, x, 8, 3, W_PER_CHANNEL_SYM, 8)
    np.testing.assert_array_equal(y, yo.astype(np.float32))


@pytest.mark.parametrize("opt", [{"convw_lock": 1}, {"convw_no_kym": 1}, {"convw_mc": 2}, {"convw_tr": 2}])
def test_convw_issue_options_are_bit_identical(opt):
    """kan_convw's issue / ring variants (lockstep rings with one commit per K
    block, one MMA per tap instead of the ky-merged form, weight multicast over
    CTA pairs, fewer rows per tile) compute the same int32 sums: stage-1-shaped
    layers in both weight schemes, bit-identical to the default."""
    for ws, silu in ((W_PER_TENSOR_ASYM, False), (W_PER_CHANNEL_SYM, True)):
        desc = conv_desc(32, 32, 32, 32, 1, 1, 0)
        desc["layers"].append({"type": "conv", "c_in": 32, "c_out": 64, "kernel": 3, "stride": 1, "padding": 1})
        desc["layers"].append({"type": "conv", "c_in": 64, "c_out": 8, "kernel": 1, "stride": 1, "padding": 0})
        Ws, Bs = weights_for(desc, seed=31, silu=silu)
        x = np.random.default_rng(31).uniform(-1.05, 1.05, (19, 32 * 32 * 32)).astype(np.float32)
        opts = dict(mode="bspline-lut", lut_k=8, lut_h=8, bits_w=8, w_scheme=ws, silu_base=silu)
        e0 = build(desc, Ws, Bs, **opts)
        e0.set_option("record_plan", 1)
        y0 = e0.model_forward(to_dev(x)).cpu().numpy()
        assert "convw layer=1" in e0.last_plan
        e1 = build(desc, Ws, Bs, engine_options=opt, **opts)
        e1.set_option("record_plan", 1)
        y1 = e1.model_forward(to_dev(x)).cpu().numpy()
        assert "convw layer=1" in e1.last_plan
        np.testing.assert_array_equal(y0, y1)


def test_convw_single_commit_default_matches_two_commits_and_oracle(oracle):
    """128-column tiles run with one commit per K block by default (it releases
    the window slot and the weight slot), and layers of two N tiles with two
    MMA-issuing warps (even / odd accumulators); the result equals the
    two-commit and single-issuer forms, the general gather kernel and the
    oracle, bit for bit, in both weight schemes."""
    for ws, silu in ((W_PER_TENSOR_ASYM, False), (W_PER_CHANNEL_SYM, True)):
        desc = conv_desc(32, 16, 16, 32, 1, 1, 0)
        desc["layers"].append({"type": "conv", "c_in": 32, "c_out": 128, "kernel": 3, "stride": 1, "padding": 1})
        desc["layers"].append({"type": "conv", "c_in": 128, "c_out": 256, "kernel": 3, "stride": 1, "padding": 1})
        desc["layers"].append({"type": "conv", "c_in": 256, "c_out": 8, "kernel": 1, "stride": 1, "padding": 0})
        Ws, Bs = weights_for(desc, seed=37, silu=silu)
        x = np.random.default_rng(37).uniform(-1.05, 1.05, (21, 32 * 16 * 16)).astype(np.float32)
        opts = dict(mode="bspline-lut", lut_k=8, lut_h=3, bits_w=8, w_scheme=ws, silu_base=silu)
        e0 = build(desc, Ws, Bs, **opts)
        e0.set_option("record_plan", 1)
        y0 = e0.model_forward(to_dev(x)).cpu().numpy()
        assert "convw layer=1" in e0.last_plan and "convw layer=2" in e0.last_plan
        # two commits, one issuer | one commit, one issuer | two issuers on the one-N-tile layer as well
        for eo in ({"convw_lock": -1}, {"convw_dual": -1}, {"convw_dual": 1}):
            y1 = build(desc, Ws, Bs, engine_options=eo, **opts).model_forward(to_dev(x)).cpu().numpy()
            np.testing.assert_array_equal(y0, y1)
        yg = build(desc, Ws, Bs, engine_options={"no_convw": 1, "no_conv3": 1}, **opts).model_forward(to_dev(x)).cpu().numpy()
        np.testing.assert_array_equal(y0, yg)
        yo = oracle.int_model_forward(desc, Ws, Bs, x, 8, 3, ws, 8)
        np.testing.assert_array_equal(y0, yo.astype(np.float32).reshape(x.shape[0], -1))

"""GPU parity: the CUDA engine (through the C ABI) against the CPU oracle and the
reference itself, on the same seeded inputs.

Bar (BASELINE.json north_star):
  * integer LUT path: bit-exact -- lattice indices, table entries, int32
    accumulators, requantized outputs (hidden lattice levels, int8 logits) and
    the fp32 logits produced from them by the fixed fp64 epilogue;
  * fp32 Cox-de Boor path: 1e-4 relative, ||y - ref||_2 / ||ref||_2;
  * bf16 path: 1e-2 relative (same metric).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2603_17230_b200 import (  # noqa: E402
    Engine, EvalOptions, OUT_I8, W_PER_CHANNEL_SYM, W_PER_TENSOR_ASYM, lattice_thresholds)

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))
FP32_TOL = 1e-4
BF16_TOL = 1e-2


def mlp_desc(dims, G, P=3):
    return {"name": "mlp", "grid": {"intervals": G, "degree": P}, "input": [dims[0]],
            "layers": [{"type": "linear", "n_in": a, "n_out": b} for a, b in zip(dims, dims[1:])]}


def make_weights(dims, G, P=3, seed=0, std=0.1, silu=False):
    rng = np.random.default_rng(seed)
    Ws, Bs = [], []
    for a, b in zip(dims, dims[1:]):
        Ws.append(rng.normal(0, std, (a * (G + P), b)))
        Bs.append(rng.normal(0, 1 / np.sqrt(a), (a, b)) if silu else None)
    return Ws, Bs


def build(dims, G, Ws, Bs, engine_options=None, **opts):
    e = Engine(mlp_desc(dims, G), 0)
    for i, (w, b) in enumerate(zip(Ws, Bs)):
        e.set_coeffs(i, w, b)
    for k, v in (engine_options or {}).items():
        e.set_option(k, v)
    e.configure(EvalOptions(**opts))
    return e


def oracle_int_model(o, G, k, h, wscheme, bits_w, Ws, Bs, x, P=3):
    """Oracle chain of the integer LUT path: levels -> int layer -> fp64 requant -> ..."""
    g = o.grid(G, P)
    lv = o.levels(g, k, x)
    level_of = np.vectorize(lambda v: o.level_of(g, k, float(v)), otypes=[np.uint16])
    ys = []
    for i, (w, b) in enumerate(zip(Ws, Bs)):
        d = o.int_layer(g, k, h, wscheme, bits_w, w, b)
        y = o.int_layer_forward(g, k, h, d, lv, w.shape[1])
        ys.append(y)
        if i + 1 < len(Ws):
            lv = level_of(y)
    return ys


def rel_err(a, b):
    """Norm-relative error ||a - b||_2 / ||b||_2 over the whole output (element-wise
    relative error is meaningless near zero outputs)."""
    a = np.asarray(a, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def to_dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


# ---------------------------------------------------------------------------------
@pytest.mark.parametrize("G,k", [(5, 8), (10, 8), (5, 4), (5, 3), (5, 2), (3, 4)])
def test_lattice_levels_bit_exact(oracle, G, k):
    x = GOLD["levels_x"]
    thr = lattice_thresholds(G, 3, k)[1:-1]
    xs = np.concatenate([x, thr, np.nextafter(thr, np.float32(-np.inf)),
                         np.nextafter(thr, np.float32(np.inf)),
                         np.random.default_rng(k).uniform(-1.2, 1.2, 300000).astype(np.float32)])
    e = build([8, 4], G, *make_weights([8, 4], G), mode="bspline-lut", lut_k=k, lut_h=8)
    got = e.layer_levels(0, to_dev(xs)).cpu().numpy().astype(np.uint16)
    np.testing.assert_array_equal(got[:len(x)], GOLD[f"levels_G{G}_k{k}"])  # reference golden
    np.testing.assert_array_equal(got, oracle.levels(oracle.grid(G, 3), k, xs))


def test_table_entries_match_reference_golden():
    for (k, h) in ((8, 8), (4, 4), (3, 3), (8, 3)):
        e = build([8, 4], 5, *make_weights([8, 4], 5), mode="bspline-lut", lut_k=k, lut_h=h)
        np.testing.assert_array_equal(e.lut(), GOLD[f"lut_P3_k{k}_h{h}"])


ACC_CASES = [
    # G, k, h, wscheme, bits_w, silu, M, n_in, N, split
    (5, 8, 8, W_PER_CHANNEL_SYM, 8, False, 200, 784, 64, 0),
    (5, 8, 8, W_PER_CHANNEL_SYM, 8, True, 200, 784, 64, 0),
    (5, 8, 8, W_PER_TENSOR_ASYM, 8, False, 300, 784, 64, 0),
    (5, 8, 8, W_PER_TENSOR_ASYM, 8, False, 129, 100, 10, 1),
    (5, 4, 4, W_PER_CHANNEL_SYM, 4, True, 257, 130, 40, 3),
    (5, 3, 3, W_PER_CHANNEL_SYM, 8, True, 64, 64, 10, 0),
    (5, 2, 2, W_PER_CHANNEL_SYM, 4, False, 1, 33, 17, 0),
    (10, 8, 8, W_PER_CHANNEL_SYM, 8, False, 130, 300, 300, 0),
    (10, 8, 8, W_PER_CHANNEL_SYM, 8, True, 130, 300, 520, 2),
    (10, 8, 8, W_PER_TENSOR_ASYM, 8, False, 64, 256, 96, 0),
    (3, 4, 8, W_PER_TENSOR_ASYM, 8, False, 100, 49, 33, 0),
]


@pytest.mark.parametrize("G,k,h,ws,bw,silu,M,n_in,N,split", ACC_CASES)
def test_int32_accumulators_bit_exact(oracle, G, k, h, ws, bw, silu, M, n_in, N, split):
    rng = np.random.default_rng(M + n_in + N)
    Ws, Bs = make_weights([n_in, N], G, seed=n_in, silu=silu)
    e = build([n_in, N], G, Ws, Bs, mode="bspline-lut", lut_k=k, lut_h=h, bits_w=bw, w_scheme=ws,
              silu_base=silu, split_k=split)
    x = rng.uniform(-1.1, 1.1, (M, n_in)).astype(np.float32)
    g = oracle.grid(G, 3)
    lv = oracle.levels(g, k, x)
    acc_s, acc_b = e.layer_accumulators(0, torch.from_numpy(lv.astype(np.int16)).cuda())
    d = oracle.int_layer(g, k, h, ws, bw, Ws[0], Bs[0])
    ws_, wb_, _ = oracle.int_accumulate(g, k, d, lv, N)
    # one int32 accumulator holds spline + SiLU-base terms (joint channel scale)
    np.testing.assert_array_equal(acc_s.cpu().numpy(), ws_)
    # the full layer from fp32 activations: fp32 logits bit-exact
    y = e.model_forward(to_dev(x)).cpu().numpy()
    yo = oracle.int_layer_forward(g, k, h, d, lv, N).astype(np.float32)
    np.testing.assert_array_equal(y, yo)


@pytest.mark.parametrize("silu", [False, True])
@pytest.mark.parametrize("bw", [8, 4])
@pytest.mark.parametrize("kh", [(8, 8), (4, 4), (3, 3), (2, 2)])
def test_c2_mlp_requantized_bit_exact(oracle, silu, bw, kh):
    """Config 2: KAN MLP [784,64,10], G=5, batch 4096, table/input precision
    sweep, int8/int4 per-channel weights, hidden outputs requantized to the next
    lattice and logits requantized to int8."""
    k, h = kh
    dims, G, M = [784, 64, 10], 5, 4096
    Ws, Bs = make_weights(dims, G, seed=2, silu=silu)
    x = np.random.default_rng(2).uniform(-1, 1, (M, 784)).astype(np.float32)
    ys = oracle_int_model(oracle, G, k, h, W_PER_CHANNEL_SYM, bw, Ws, Bs, x)
    s_out = float(np.abs(ys[-1]).max() / 127)
    e = build(dims, G, Ws, Bs, mode="bspline-lut", lut_k=k, lut_h=h, bits_w=bw,
              w_scheme=W_PER_CHANNEL_SYM, silu_base=silu)
    y = e.model_forward(to_dev(x)).cpu().numpy()
    np.testing.assert_array_equal(y, ys[-1].astype(np.float32))
    e.configure(EvalOptions(mode="bspline-lut", lut_k=k, lut_h=h, bits_w=bw,
                            w_scheme=W_PER_CHANNEL_SYM, silu_base=silu, out_kind=OUT_I8,
                            out_scale=s_out))
    q = e.model_forward(to_dev(x)).cpu().numpy()
    np.testing.assert_array_equal(q, oracle.requant_i8(ys[-1], s_out))


def test_reference_mode_matches_tabulated_kan_forward(oracle, ref):
    """The reference's own scheme (per-tensor asymmetric u8 W, no SiLU):
    GPU logits == integer restatement (bit-exact in fp32) and == the
    reference's fp64 tabulated_kan_forward within fp32 rounding."""
    G, k, h = 5, 8, 8
    rng = np.random.default_rng(9)
    x = rng.uniform(-1, 1, (1024, 784)).astype(np.float32)
    W = rng.normal(0, 0.1, (784 * 8, 10))
    e = build([784, 10], G, [W], [None], mode="bspline-lut", lut_k=k, lut_h=h, bits_w=8,
              w_scheme=W_PER_TENSOR_ASYM)
    y = e.model_forward(to_dev(x)).cpu().numpy()
    g = oracle.grid(G, 3)
    d = oracle.int_layer(g, k, h, 0, 8, W)
    yo = oracle.int_layer_forward(g, k, h, d, oracle.levels(g, k, x), 10)
    np.testing.assert_array_equal(y, yo.astype(np.float32))
    r = ref.lut_forward(G, 3, k, h, 8, x.astype(np.float64), W)
    assert rel_err(y, r) < 1e-6
    # argmax parity with the reference's predict (acceptance.cpp:259-294)
    assert (e.predict(to_dev(x)).cpu().numpy() == r.argmax(1)).mean() > 0.999


@pytest.mark.parametrize("dims,G", [([784, 64, 10], 5), ([300, 100, 10], 10), ([49, 33], 3)])
def test_fp32_cox_de_boor_path(oracle, ref, dims, G):
    Ws, _ = make_weights(dims, G, seed=4)
    x = np.random.default_rng(4).uniform(-1.1, 1.1, (777, dims[0])).astype(np.float32)
    e = build(dims, G, Ws, [None] * len(Ws), mode="fp32")
    y = e.model_forward(to_dev(x)).cpu().numpy()
    r = x.astype(np.float64)
    for w in Ws:
        r = ref.linear_forward(G, 3, r, w)
    assert rel_err(y, r) < FP32_TOL


@pytest.mark.parametrize("dims,G", [([784, 64], 5), ([300, 100], 10), ([3072, 256], 10),
                                    ([64, 10], 5)])
def test_bf16_layer(oracle, dims, G):
    """One KAN layer on the bf16 tensor-core path vs the fp64 reference: 1e-2."""
    Ws, _ = make_weights(dims, G, seed=6)
    x = np.random.default_rng(6).uniform(-1.1, 1.1, (1000, dims[0])).astype(np.float32)
    e = build(dims, G, Ws, [None] * len(Ws), mode="bf16")
    y = e.model_forward(to_dev(x)).cpu().numpy()
    r = oracle.linear_forward(oracle.grid(G, 3), x.astype(np.float64), Ws[0])
    assert rel_err(y, r) < BF16_TOL


@pytest.mark.parametrize("dims,G", [([784, 64, 10], 5), ([300, 100, 10], 10)])
def test_bf16_model(oracle, dims, G):
    """Stacked bf16 layers: the per-layer bf16 rounding of basis and weights is
    amplified by the next layer's steep basis (knot spacing 2/G), so the model
    bound is the per-layer 1e-2 times the layer count, plus argmax agreement."""
    Ws, _ = make_weights(dims, G, seed=6)
    x = np.random.default_rng(6).uniform(-1, 1, (1000, dims[0])).astype(np.float32)
    e = build(dims, G, Ws, [None] * len(Ws), mode="bf16")
    y = e.model_forward(to_dev(x)).cpu().numpy()
    g = oracle.grid(G, 3)
    r = x.astype(np.float64)
    for w in Ws:
        r = oracle.linear_forward(g, r, w)
    assert rel_err(y, r) < BF16_TOL * len(Ws)
    assert (y.argmax(1) == r.argmax(1)).mean() > 0.97


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_float_paths_with_silu_base(oracle, mode):
    dims, G = [256, 48, 10], 5
    Ws, Bs = make_weights(dims, G, seed=8, silu=True)
    x = np.random.default_rng(8).uniform(-1, 1, (500, 256)).astype(np.float32)
    e = build(dims, G, Ws, Bs, mode=mode, silu_base=True)
    y = e.model_forward(to_dev(x)).cpu().numpy()
    g = oracle.grid(G, 3)
    r = x.astype(np.float64)
    for w, b in zip(Ws, Bs):
        xc = np.vectorize(lambda v: oracle.lib.kor_clamp(g, float(v)))(r)
        r = oracle.linear_forward(g, r, w) + (xc / (1 + np.exp(-xc))) @ b
    assert rel_err(y, r) < (FP32_TOL if mode == "fp32" else BF16_TOL)


def test_empty_and_ragged_batches(oracle):
    dims, G = [784, 64, 10], 5
    Ws, Bs = make_weights(dims, G, seed=3, silu=True)
    e = build(dims, G, Ws, Bs, mode="bspline-lut", silu_base=True)
    out = e.model_forward(torch.empty((0, 784), device="cuda"))
    assert out.shape == (0, 10)
    x = np.random.default_rng(3).uniform(-1, 1, (333, 784)).astype(np.float32)
    full = e.model_forward(to_dev(x)).cpu().numpy()
    for m in (1, 7, 128, 129):
        np.testing.assert_array_equal(e.model_forward(to_dev(x[:m])).cpu().numpy(), full[:m])


def test_split_k_invariance_and_row_independence_at_c3_shape():
    """Config 3 layer 1 at full width (G=10, 3072 -> 1024): the int32 result is
    independent of the K split and rows are independent (size-independent
    properties standing in for the oracle at full batch)."""
    G, M = 10, 2048
    Ws, Bs = make_weights([3072, 1024], G, seed=12, std=0.05)
    x = to_dev(np.random.default_rng(12).uniform(-1, 1, (M, 3072)))
    outs = []
    for split in (1, 3, 8):
        e = build([3072, 1024], G, Ws, Bs, mode="bspline-lut", split_k=split)
        outs.append(e.model_forward(x).cpu().numpy())
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[0], outs[2])
    perm = torch.randperm(M, device="cuda")
    y2 = e.model_forward(x[perm].contiguous()).cpu().numpy()
    np.testing.assert_array_equal(y2, outs[0][perm.cpu().numpy()])


def test_c3_layer_rows_bit_exact(oracle):
    G, k, h = 10, 8, 8
    Ws, _ = make_weights([3072, 1024], G, seed=13, std=0.05)
    x = np.random.default_rng(13).uniform(-1, 1, (40, 3072)).astype(np.float32)
    e = build([3072, 1024], G, Ws, [None], mode="bspline-lut")
    y = e.model_forward(to_dev(x)).cpu().numpy()
    g = oracle.grid(G, 3)
    d = oracle.int_layer(g, k, h, W_PER_CHANNEL_SYM, 8, Ws[0])
    np.testing.assert_array_equal(y, oracle.int_layer_forward(g, k, h, d, oracle.levels(g, k, x),
                                                              1024).astype(np.float32))


def test_forward_host_equals_device_path():
    dims, G = [784, 64, 10], 5
    Ws, Bs = make_weights(dims, G, seed=5, silu=True)
    e = build(dims, G, Ws, Bs, mode="bspline-lut", silu_base=True)
    x = np.random.default_rng(5).uniform(-1, 1, (1024, 784)).astype(np.float32)
    np.testing.assert_array_equal(e.forward_host(x), e.model_forward(to_dev(x)).cpu().numpy())
    # the 64 -> 10 output layer runs inside layer 0's split-K launch
    assert e.last_launches == 1


@pytest.mark.parametrize("M", [4096, 1024, 300, 12800])
def test_fused_output_layer_matches_separate_launches(oracle, M):
    """The small output layer runs inside the previous layer's launch: in the
    split-K reduction (auto split: 4, 8, 8 and 2 CTAs per tile here), or after
    each tile's epilogue of a persistent launch (split_k=1 with option
    fuse_persistent).  By default a persistent launch leaves it to its own kernel.  All are the same integer computation:
    bit-identical logits, and equal to the oracle."""
    dims, G = [784, 64, 10], 5
    Ws, Bs = make_weights(dims, G, seed=6, silu=True)
    x = np.random.default_rng(M).uniform(-1, 1, (M, 784)).astype(np.float32)
    fused = build(dims, G, Ws, Bs, mode="bspline-lut", silu_base=True)
    yf = fused.model_forward(to_dev(x)).cpu().numpy()
    assert fused.last_launches == 1
    pers = build(dims, G, Ws, Bs, engine_options={"fuse_persistent": 1}, mode="bspline-lut", silu_base=True, split_k=1)
    yp = pers.model_forward(to_dev(x)).cpu().numpy()
    assert pers.last_launches == 1
    np.testing.assert_array_equal(yf, yp)
    sep = build(dims, G, Ws, Bs, mode="bspline-lut", silu_base=True, split_k=1)
    ys = sep.model_forward(to_dev(x)).cpu().numpy()
    assert sep.last_launches == 2
    np.testing.assert_array_equal(yf, ys)
    yo = oracle_int_model(oracle, G, 8, 8, W_PER_CHANNEL_SYM, 8, Ws, Bs, x)[-1]
    np.testing.assert_array_equal(yf, yo.astype(np.float32))


def test_fused_output_layer_many_tiles_per_cta(oracle):
    """Persistent fused launch with more tiles than SMs (several tiles per CTA,
    the hidden-level buffer reused tile after tile), int8 logits, ragged batch."""
    dims, G = [96, 48, 12], 5
    Ws, Bs = make_weights(dims, G, seed=16, silu=True)
    M = 128 * 300 + 77
    x = np.random.default_rng(M).uniform(-1.05, 1.05, (M, 96)).astype(np.float32)
    opts = dict(mode="bspline-lut", silu_base=True, out_kind=OUT_I8, out_scale=0.05)
    e = build(dims, G, Ws, Bs, engine_options={"fuse_persistent": 1}, **opts)
    y = e.model_forward(to_dev(x)).cpu().numpy()
    assert e.last_launches == 1
    ys = build(dims, G, Ws, Bs, **opts).model_forward(to_dev(x)).cpu().numpy()
    np.testing.assert_array_equal(y, ys)


def test_level_prepass_matches_in_kernel_levels(oracle):
    """Large fp32-input layers take an HBM-bound level prepass and the GEMM
    reads u16 levels; the result is bit-identical to computing the levels in
    the producers (threshold lowered here to exercise it at test size)."""
    dims, G = [300, 100, 10], 10
    Ws, Bs = make_weights(dims, G, seed=8, silu=True)
    x = np.random.default_rng(8).uniform(-1.1, 1.1, (1000, 300)).astype(np.float32)
    opts = dict(mode="bspline-lut", lut_k=8, lut_h=8, silu_base=True, split_k=1)
    y0 = build(dims, G, Ws, Bs, **opts).model_forward(to_dev(x)).cpu().numpy()
    e = build(dims, G, Ws, Bs, engine_options={"level_prepass_min": 0}, **opts)
    y1 = e.model_forward(to_dev(x)).cpu().numpy()
    assert e.last_launches == 3  # prepass + layer 0 + small output layer
    np.testing.assert_array_equal(y0, y1)
    yo = oracle_int_model(oracle, G, 8, 8, W_PER_CHANNEL_SYM, 8, Ws, Bs, x)[-1]
    np.testing.assert_array_equal(y1, yo.astype(np.float32))


@pytest.mark.parametrize("name", ["lekan", "cnn3"])
def test_fp32_conv_models_match_reference(ref, name):
    """EvalMode::kFp32 on the reference's conv descriptors (convkan_forward with
    RecursiveBasis, maxpool2, flatten): fp32 im2col rows through the fp32
    Cox-de Boor kernel, within the fp32 bar."""
    import json as _json
    desc = {"lekan": {"name": "LeKAN", "grid": {"intervals": 3, "degree": 3}, "input": [1, 28, 28],
                      "layers": [{"type": "conv", "c_in": 1, "c_out": 6, "kernel": 5, "stride": 1, "padding": 0},
                                 {"type": "maxpool", "window": 2},
                                 {"type": "conv", "c_in": 6, "c_out": 16, "kernel": 5, "stride": 1, "padding": 2},
                                 {"type": "maxpool", "window": 2}, {"type": "flatten"},
                                 {"type": "linear", "n_in": 576, "n_out": 10}]},
            "cnn3": {"name": "c", "grid": {"intervals": 5, "degree": 3}, "input": [3, 17, 17],
                     "layers": [{"type": "conv", "c_in": 3, "c_out": 8, "kernel": 3, "stride": 1, "padding": 1},
                                {"type": "conv", "c_in": 8, "c_out": 12, "kernel": 3, "stride": 2, "padding": 1},
                                {"type": "maxpool", "window": 2}, {"type": "flatten"},
                                {"type": "linear", "n_in": 192, "n_out": 10}]}}[name]
    nb = desc["grid"]["intervals"] + desc["grid"]["degree"]
    rng = np.random.default_rng(7)
    Ws = []
    for l in desc["layers"]:
        if l["type"] == "conv":
            Ws.append(rng.normal(0, 0.1, (l["c_in"] * l["kernel"] ** 2 * nb, l["c_out"])))
        elif l["type"] == "linear":
            Ws.append(rng.normal(0, 0.1, (l["n_in"] * nb, l["n_out"])))
    e = Engine(desc, 0)
    for i, w in enumerate(Ws):
        e.set_coeffs(i, w)
    e.configure(EvalOptions(mode="fp32"))
    D = int(np.prod(desc["input"]))
    x = rng.uniform(-1, 1, (9, D)).astype(np.float32)
    y = e.model_forward(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
    r = ref.model_forward(_json.dumps(desc), Ws, x.astype(np.float64), 10, mode=0)
    assert np.linalg.norm(y - r) / np.linalg.norm(r) < FP32_TOL
    assert np.array_equal(e.predict(torch.from_numpy(x).cuda()).cpu().numpy(), r.argmax(1))


@pytest.mark.parametrize("dims", [[200, 64], [120, 96, 128], [150, 80], [100, 300]])
@pytest.mark.parametrize("silu", [False, True])
@pytest.mark.parametrize("split", [1, 0])
def test_fp32_output_epilogue_paths_bit_exact(oracle, dims, silu, split):
    """fp32 row-major outputs: full-width column tiles take the straight-line
    epilogue staged through shared memory (kan_gemm.cu, FE instantiation),
    ragged ones (N = 300: a 256 + 44 column split) and split-K launches take
    finish4.  M = 333 leaves a partial row tile.  All are bit-exact with the
    oracle and identical with the staging switched off (option epi_stage=0)."""
    G, M = 5, 333
    Ws, Bs = make_weights(dims, G, seed=11, silu=silu)
    x = np.random.default_rng(11).uniform(-1.05, 1.05, (M, dims[0])).astype(np.float32)
    opts = dict(mode="bspline-lut", lut_k=8, lut_h=8, silu_base=silu, split_k=split)
    y = build(dims, G, Ws, Bs, **opts).model_forward(to_dev(x)).cpu().numpy()
    yo = oracle_int_model(oracle, G, 8, 8, W_PER_CHANNEL_SYM, 8, Ws, Bs, x)[-1]
    np.testing.assert_array_equal(y, yo.astype(np.float32))
    y0 = build(dims, G, Ws, Bs, engine_options={"epi_stage": 0}, **opts).model_forward(to_dev(x)).cpu().numpy()
    np.testing.assert_array_equal(y0, y)

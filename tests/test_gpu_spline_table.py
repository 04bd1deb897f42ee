"""GPU parity of spline-table mode (EvalMode::kSplineTable, spline_table.hpp)
through the C ABI, against the oracle restatement (pinned to the reference in
test_spline_table_cpu.py).  Bar: bit-exact -- table entries and quantizers,
input levels, integer sums, hidden levels, and the fp32 outputs (the fp64
s_out * sum rounded once to fp32)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2603_17230_b200 import (  # noqa: E402
    Engine, EvalOptions, build_spline_tables, spline_table_forward, spline_thresholds)


def mlp_desc(dims, G=5, P=3):
    return {"name": "mlp", "grid": {"intervals": G, "degree": P}, "input": [dims[0]],
            "layers": [{"type": "linear", "n_in": a, "n_out": b} for a, b in zip(dims, dims[1:])]}


def st_engine(desc, Ws, bits_a, h):
    e = Engine(desc, 0)
    for i, w in enumerate(Ws):
        e.set_coeffs(i, w)
    e.configure(EvalOptions(mode="spline-table", lut_k=bits_a, lut_h=h))
    return e


@pytest.mark.parametrize("n_in,n_out,bits_a,h", [(7, 5, 8, 8), (13, 3, 4, 6), (3, 2, 1, 2),
                                                 (20, 9, 5, 7), (64, 10, 8, 8), (40, 48, 3, 3),
                                                 (33, 130, 6, 5)])
def test_tables_bit_exact(oracle, n_in, n_out, bits_a, h):
    rng = np.random.default_rng(n_in + 7 * bits_a)
    W = rng.normal(0, 0.1, (n_in * 8, n_out))
    got = build_spline_tables(W, n_in, n_out, 5, 3, bits_a, h)
    want = oracle.spline_tables(oracle.grid(5, 3), W, n_in, n_out, bits_a, h)
    np.testing.assert_array_equal(got["values"], want["values"])
    np.testing.assert_array_equal(got["qp_d"], want["qp_d"])
    np.testing.assert_array_equal(got["qp_i"], want["qp_i"])


def test_zero_coefficient_tables(oracle):
    W = np.zeros((3 * 8, 2))
    got = build_spline_tables(W, 3, 2, 5, 3, 4, 8)
    want = oracle.spline_tables(oracle.grid(5, 3), W, 3, 2, 4, 8)
    np.testing.assert_array_equal(got["values"], want["values"])
    np.testing.assert_array_equal(got["qp_d"], want["qp_d"])


@pytest.mark.parametrize("bits_a", [1, 3, 8])
def test_input_levels_bit_exact(oracle, bits_a):
    e = st_engine(mlp_desc([4, 2]), [np.random.default_rng(0).normal(0, 0.1, (32, 2))], bits_a, 8)
    thr = spline_thresholds(bits_a)
    rng = np.random.default_rng(bits_a)
    x = np.concatenate([rng.uniform(-1.5, 1.5, 100000).astype(np.float32), thr[1:],
                        np.nextafter(thr[1:], np.float32(-np.inf)),
                        np.array([0.0, -0.0, 50.0, -50.0, 1e30, np.inf, -np.inf, np.nan], np.float32)])
    got = e.layer_levels(0, torch.from_numpy(x).cuda()).cpu().numpy().astype(np.int64)
    s, z, qh = oracle.quant_params(-1.0, 1.0, bits_a)
    want = np.array([oracle.lib.kor_spline_level(float(v), s, z, qh) for v in x])
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("n_in,n_out,bits_a", [(784, 64, 8), (64, 10, 8), (300, 33, 4), (1000, 600, 2)])
def test_integer_sums_bit_exact(oracle, n_in, n_out, bits_a):
    rng = np.random.default_rng(n_in)
    W = rng.normal(0, 0.1, (n_in * 8, n_out))
    e = st_engine(mlp_desc([n_in, n_out]), [W], bits_a, 8)
    t = e.spline_table(0)
    M = 77
    lv = rng.integers(0, 1 << bits_a, (M, n_in)).astype(np.uint16)
    acc, _ = e.layer_accumulators(0, torch.from_numpy(lv.astype(np.int16)).cuda())
    want = oracle.spline_accumulate(t, lv.astype(np.uint8))
    np.testing.assert_array_equal(acc.cpu().numpy().astype(np.int64), want)


@pytest.mark.parametrize("dims,M,bits_a,h", [([784, 64, 10], 1024, 8, 8), ([784, 64, 10], 300, 4, 4),
                                             ([784, 64, 10], 257, 2, 2), ([40, 24, 10], 1, 8, 8),
                                             ([50, 1030, 7], 40, 5, 6), ([3, 17, 5, 2], 129, 3, 3)])
def test_mlp_forward_bit_exact(oracle, dims, M, bits_a, h):
    rng = np.random.default_rng(M)
    Ws = [rng.normal(0, 0.1, (a * 8, b)) for a, b in zip(dims, dims[1:])]
    desc = mlp_desc(dims)
    e = st_engine(desc, Ws, bits_a, h)
    x = rng.uniform(-1, 1, (M, dims[0])).astype(np.float32)
    x[0, :3] = [50.0, -50.0, 0.0]
    y = e.model_forward(torch.from_numpy(x).cuda()).cpu().numpy()
    tabs = oracle.spline_model_tables(desc, Ws, bits_a, h)
    want = oracle.spline_model_forward(desc, tabs, x.astype(np.float64)).astype(np.float32)
    np.testing.assert_array_equal(y, want)
    np.testing.assert_array_equal(e.forward_host(x), want)
    fused = len(Ws) >= 2 and dims[-1] <= 16 and dims[-2] <= 512  # output layer runs fused
    assert e.last_launches == len(Ws) - int(fused) + 1  # + the input-level prepass


def test_conv_models_bit_exact(oracle):
    """LeKAN (conv, maxpool, flatten, linear) and a padded 3x3 conv stack."""
    rng = np.random.default_rng(0)
    lekan = {"name": "LeKAN", "grid": {"intervals": 3, "degree": 3}, "input": [1, 28, 28],
             "layers": [{"type": "conv", "c_in": 1, "c_out": 6, "kernel": 5, "stride": 1, "padding": 0},
                        {"type": "maxpool", "window": 2},
                        {"type": "conv", "c_in": 6, "c_out": 16, "kernel": 5, "stride": 1, "padding": 0},
                        {"type": "maxpool", "window": 2}, {"type": "flatten"},
                        {"type": "linear", "n_in": 256, "n_out": 10}]}
    Ws = [rng.normal(0, 0.1, (25 * 6, 6)), rng.normal(0, 0.1, (150 * 6, 16)),
          rng.normal(0, 0.1, (256 * 6, 10))]
    x = rng.uniform(-1, 1, (37, 784)).astype(np.float32)
    for bits_a, h in ((8, 8), (6, 7), (3, 4)):
        e = st_engine(lekan, Ws, bits_a, h)
        y = e.model_forward(torch.from_numpy(x).cuda()).cpu().numpy()
        tabs = oracle.spline_model_tables(lekan, Ws, bits_a, h)
        want = oracle.spline_model_forward(lekan, tabs, x.astype(np.float64)).astype(np.float32)
        np.testing.assert_array_equal(y, want)
    conv = {"name": "c", "grid": {"intervals": 5, "degree": 3}, "input": [16, 13, 13],
            "layers": [{"type": "conv", "c_in": 16, "c_out": 20, "kernel": 3, "stride": 1, "padding": 1},
                       {"type": "conv", "c_in": 20, "c_out": 24, "kernel": 3, "stride": 2, "padding": 1}]}
    Ws = [rng.normal(0, 0.05, (16 * 9 * 8, 20)), rng.normal(0, 0.05, (20 * 9 * 8, 24))]
    e = st_engine(conv, Ws, 8, 8)
    x = rng.uniform(-1, 1, (5, 16 * 169)).astype(np.float32)
    y = e.model_forward(torch.from_numpy(x).cuda()).cpu().numpy()
    tabs = oracle.spline_model_tables(conv, Ws, 8, 8)
    want = oracle.spline_model_forward(conv, tabs, x.astype(np.float64)).reshape(5, -1)
    np.testing.assert_array_equal(y, want.astype(np.float32))


def test_c4_shaped_conv_bit_exact(oracle):
    rng = np.random.default_rng(4)
    desc = {"name": "c4", "grid": {"intervals": 5, "degree": 3}, "input": [64, 32, 32],
            "layers": [{"type": "conv", "c_in": 64, "c_out": 64, "kernel": 3, "stride": 1, "padding": 1}]}
    W = rng.normal(0, 0.05, (64 * 9 * 8, 64))
    e = st_engine(desc, [W], 8, 8)
    x = rng.uniform(-1, 1, (2, 64 * 1024)).astype(np.float32)
    y = e.model_forward(torch.from_numpy(x).cuda()).cpu().numpy()
    tabs = oracle.spline_model_tables(desc, [W], 8, 8)
    want = oracle.spline_model_forward(desc, tabs, x.astype(np.float64)).reshape(2, -1)
    np.testing.assert_array_equal(y, want.astype(np.float32))


def test_supplied_tables_match_built_tables_and_reference_forward(oracle, ref):
    """EvalOptions::tables supplied by the caller (a table set the reference
    itself built) run through spline_table_forward unchanged."""
    rng = np.random.default_rng(2)
    n_in, n_out = 100, 12
    W = rng.normal(0, 0.1, (n_in * 8, n_out))
    t = ref.spline_tables(5, 3, W, n_in, n_out, 6, 7)
    x = rng.uniform(-1.2, 1.2, (333, n_in)).astype(np.float32)
    got = spline_table_forward(torch.from_numpy(x).cuda(), t).cpu().numpy()
    want = ref.spline_forward(t, x.astype(np.float64)).astype(np.float32)
    np.testing.assert_array_equal(got, want)
    e = st_engine(mlp_desc([n_in, n_out]), [W], 6, 7)
    np.testing.assert_array_equal(e.model_forward(torch.from_numpy(x).cuda()).cpu().numpy(), want)


def test_empty_batch_and_errors():
    rng = np.random.default_rng(1)
    e = st_engine(mlp_desc([16, 8]), [rng.normal(0, 0.1, (128, 8))], 8, 8)
    y = e.model_forward(torch.zeros((0, 16), device="cuda"))
    assert y.shape == (0, 8)
    with pytest.raises(ValueError):
        st_engine(mlp_desc([16, 8]), [rng.normal(0, 0.1, (128, 8))], 9, 8)
    with pytest.raises(ValueError):
        st_engine(mlp_desc([16, 8]), [rng.normal(0, 0.1, (128, 8))], 4, 1)
    with pytest.raises(ValueError):
        spline_table_forward(torch.zeros((2, 5), device="cuda"),
                             build_spline_tables(rng.normal(0, 0.1, (32, 2)), 4, 2, 5, 3, 4, 8))

"""Spline-table mode (spline_table.hpp), CPU side: the oracle restatement
pinned against the reference (live, oracle/_ref) and against the reference's
own known answers (proj/tests/test_spline_table.cpp), and the engine's host
rule for fp32 input levels (exact thresholds) against quantize_value."""
import json

import numpy as np
import pytest

G, P = 5, 3


def _coeffs(rng, n_in, n_out, G=G, P=P, std=0.1):
    return rng.normal(0, std, (n_in * (G + P), n_out))


@pytest.mark.parametrize("n_in,n_out,bits_a,h", [(7, 5, 8, 8), (13, 3, 4, 6), (3, 2, 1, 2),
                                                 (20, 9, 5, 7), (33, 17, 3, 3)])
def test_oracle_tables_and_forward_match_reference(oracle, ref, n_in, n_out, bits_a, h):
    rng = np.random.default_rng(n_in * 100 + bits_a)
    W = _coeffs(rng, n_in, n_out)
    a = oracle.spline_tables(oracle.grid(G, P), W, n_in, n_out, bits_a, h)
    b = ref.spline_tables(G, P, W, n_in, n_out, bits_a, h)
    np.testing.assert_array_equal(a["values"], b["values"])
    np.testing.assert_array_equal(a["qp_d"], b["qp_d"])
    np.testing.assert_array_equal(a["qp_i"], b["qp_i"])
    x = rng.uniform(-1.3, 1.3, (64, n_in))
    x[0] = 0.0
    x[1, :] = 50.0
    np.testing.assert_array_equal(oracle.spline_forward(a, x), ref.spline_forward(b, x))


def test_oracle_conv_tables_match_reference(oracle, ref):
    rng = np.random.default_rng(5)
    W = _coeffs(rng, 2 * 9, 3)
    a = oracle.spline_tables(oracle.grid(G, P), W, 18, 3, 5, 7)
    b = ref.spline_tables(G, P, W, 2, 3, 5, 7, kernel=3, stride=1, padding=1)
    np.testing.assert_array_equal(a["values"], b["values"])
    assert b["stored_bits"] == 18 * 3 * 32 * 7


def test_known_answers_from_reference_tests(oracle):
    """test_spline_table.cpp:22-62: zero coefficients tabulate to exact zeros,
    the stored-bits closed form, conv table count, single-connection lookups."""
    g3 = oracle.grid(3, 3)
    t = oracle.spline_tables(g3, np.zeros((3 * 6, 2)), 3, 2, 4, 8)
    s, z = t["qp_d"][1], t["qp_i"][2]
    assert np.all(s * (t["values"].astype(np.int64) - z) == 0.0)
    wide = oracle.spline_tables(g3, np.zeros((784 * 6, 10)), 784, 10, 8, 8)
    assert wide["values"].size * 8 == 16056320
    narrow = oracle.spline_tables(g3, np.zeros((784 * 6, 10)), 784, 10, 4, 6)
    assert narrow["values"].size * 6 == 752640
    conv = oracle.spline_tables(g3, np.zeros((5 * 5 * 3 * 6, 4)), 5 * 5 * 3, 4, 3, 4)
    assert conv["values"].shape == (75, 4, 8)
    rng = np.random.default_rng(3)
    one = oracle.spline_tables(g3, rng.uniform(-1, 1, (6, 1)), 1, 1, 5, 8)
    for m in range(0, 32, 5):
        x = one["qp_d"][0] * (m - one["qp_i"][0])  # dequantize_value(m, in_qp)
        y = oracle.spline_forward(one, np.array([[x]]))
        assert y[0, 0] == one["qp_d"][1] * (int(one["values"][0, 0, m]) - one["qp_i"][2])


def test_out_of_range_inputs_clamp_like_the_edge_levels(oracle):
    """test_spline_table.cpp:109-129."""
    g3 = oracle.grid(3, 3)
    rng = np.random.default_rng(9)
    t = oracle.spline_tables(g3, rng.uniform(-1, 1, (4 * 6, 2)), 4, 2, 4, 8)
    s, z, qh = t["qp_d"][0], t["qp_i"][0], t["qp_i"][1]
    out = oracle.spline_forward(t, np.array([[-50.0, 50.0, 0.0, 1e9]]))
    edge = oracle.spline_forward(t, np.array([[s * (0 - z), s * (qh - z), 0.0, s * (qh - z)]]))
    assert np.all(np.isfinite(out))
    np.testing.assert_array_equal(out, edge)


def test_oracle_model_forward_matches_reference_model_forward(oracle, ref):
    """model_forward in EvalMode::kSplineTable (eval.hpp:121-127) over LeKAN
    (conv, maxpool, flatten, linear) and a 2-layer MLP."""
    rng = np.random.default_rng(0)
    lekan = {"name": "LeKAN", "grid": {"intervals": 3, "degree": 3}, "input": [1, 28, 28],
             "layers": [{"type": "conv", "c_in": 1, "c_out": 6, "kernel": 5, "stride": 1, "padding": 0},
                        {"type": "maxpool", "window": 2},
                        {"type": "conv", "c_in": 6, "c_out": 16, "kernel": 5, "stride": 1, "padding": 0},
                        {"type": "maxpool", "window": 2}, {"type": "flatten"},
                        {"type": "linear", "n_in": 256, "n_out": 10}]}
    Ws = [rng.normal(0, 0.1, (25 * 6, 6)), rng.normal(0, 0.1, (150 * 6, 16)),
          rng.normal(0, 0.1, (256 * 6, 10))]
    x = rng.uniform(-1, 1, (4, 784))
    for bits_a, h in ((6, 7), (8, 8), (2, 2)):
        tabs = oracle.spline_model_tables(lekan, Ws, bits_a, h)
        np.testing.assert_array_equal(oracle.spline_model_forward(lekan, tabs, x),
                                      ref.model_forward(json.dumps(lekan), Ws, x, 10, mode=3,
                                                        k=bits_a, h=h))
    mlp = {"name": "m", "grid": {"intervals": 5, "degree": 3}, "input": [40],
           "layers": [{"type": "linear", "n_in": 40, "n_out": 24},
                      {"type": "linear", "n_in": 24, "n_out": 10}]}
    Ws = [rng.normal(0, 0.1, (40 * 8, 24)), rng.normal(0, 0.1, (24 * 8, 10))]
    x = rng.uniform(-1, 1, (50, 40))
    tabs = oracle.spline_model_tables(mlp, Ws, 8, 8)
    np.testing.assert_array_equal(oracle.spline_model_forward(mlp, tabs, x),
                                  ref.model_forward(json.dumps(mlp), Ws, x, 10, mode=3, k=8, h=8))


def _emulate_st_level(x, thr, inv_s, zf, qhi):
    """numpy float32 replica of kan_spline_table.cu st_level_f32."""
    x = x.astype(np.float32)
    with np.errstate(invalid="ignore", over="ignore"):
        t = np.float32(x) * np.float32(inv_s) + np.float32(zf)  # fmaf: exact enough for the estimate
    t = np.where(np.isnan(t), np.float32(0), t)
    n = np.clip(np.rint(np.clip(t, -1e9, 1e9)), 0, qhi).astype(np.int64)
    down = (n > 0) & (x < thr[n])
    up = (~down) & (n < qhi) & (x >= thr[np.minimum(n + 1, qhi)])
    return np.where(x < thr[qhi + 1], n - down + up, 0)


@pytest.mark.parametrize("bits_a", [1, 2, 3, 4, 5, 7, 8])
def test_spline_level_threshold_rule_is_exact(oracle, bits_a):
    from paper_2603_17230_b200 import spline_thresholds
    thr = spline_thresholds(bits_a)
    s, z, qh = oracle.quant_params(-1.0, 1.0, bits_a)
    assert thr.size == qh + 2
    rng = np.random.default_rng(bits_a)
    xs = [rng.uniform(-1.2, 1.2, 20000).astype(np.float32),
          np.array([0.0, -0.0, 1.0, -1.0, 50.0, -50.0, 1e9, -1e9, 1e19, 1e30, -1e30, np.inf,
                    -np.inf, np.nan], np.float32)]
    fin = thr[1:]  # every level step and the llround overflow point
    xs += [fin, np.nextafter(fin, np.float32(-np.inf)), np.nextafter(fin, np.float32(np.inf))]
    x = np.concatenate(xs)
    want = np.array([oracle.lib.kor_spline_level(float(v), s, z, qh) for v in x])
    got = _emulate_st_level(x, thr, 1.0 / s, float(z), qh)
    np.testing.assert_array_equal(got, want)

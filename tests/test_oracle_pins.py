"""Pin the CPU oracle (oracle/kan_oracle.c) before trusting it.

1. Against the committed golden vectors generated from the reference itself
   (tests/golden/make_golden.py over oracle/_ref) -- runs everywhere.
2. Against the reference's own known-answer tests, restated
   (test_grid.cpp, test_quant.cpp, test_lut.cpp, test_layers.cpp).
3. Against the reference compiled from /root/reference (oracle/_ref), where
   present: exhaustive LUT equality, lattice levels, bit-exact layer forwards.
"""
import os

import numpy as np
import pytest

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))


# ---- 1. golden vectors -------------------------------------------------------------
@pytest.mark.parametrize("P", [1, 2, 3])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("h", [2, 3, 4, 8])
def test_lut_entries_match_reference_golden(oracle, P, k, h):
    np.testing.assert_array_equal(oracle.lut(P, k, h), GOLD[f"lut_P{P}_k{k}_h{h}"])


@pytest.mark.parametrize("G,k", [(5, 8), (10, 8), (5, 4), (5, 3), (5, 2), (3, 4)])
def test_lattice_levels_match_reference_golden(oracle, G, k):
    g = oracle.grid(G, 3)
    np.testing.assert_array_equal(oracle.levels(g, k, GOLD["levels_x"]), GOLD[f"levels_G{G}_k{k}"])


@pytest.mark.parametrize("G,k,h", [(5, 8, 8), (10, 8, 8), (5, 8, 3), (5, 4, 4)])
def test_every_lookup_matches_reference_golden(oracle, G, k, h):
    g = oracle.grid(G, 3)
    lut = oracle.lut(3, k, h)
    vals = GOLD[f"lookup_G{G}_k{k}_h{h}_vals"]
    start = GOLD[f"lookup_G{G}_k{k}_h{h}_start"]
    cnt = GOLD[f"lookup_G{G}_k{k}_h{h}_count"]
    for a in range((G << k) + 1):
        v, s = oracle.lut_lookup(g, k, lut, a)
        assert s == start[a] and len(v) == cnt[a]
        np.testing.assert_array_equal(v, vals[a, :cnt[a]])


def test_forwards_match_reference_golden_bit_for_bit(oracle):
    g = oracle.grid(5, 3)
    acts, coeffs = GOLD["fwd_acts"], GOLD["fwd_coeffs"]
    np.testing.assert_array_equal(oracle.linear_forward(g, acts, coeffs), GOLD["fwd_linear_G5"])
    np.testing.assert_array_equal(oracle.lut_forward(g, 8, 8, 8, acts, coeffs),
                                  GOLD["fwd_lut_G5_k8_h8_w8"])
    np.testing.assert_array_equal(oracle.lut_forward(g, 4, 4, 4, acts, coeffs),
                                  GOLD["fwd_lut_G5_k4_h4_w4"])


def test_im2col_matches_reference_golden(oracle):
    np.testing.assert_array_equal(oracle.im2col(GOLD["im2col_in"], 3, 1, 1), GOLD["im2col_k3s1p1"])


# ---- 2. the reference's known-answer tests, restated ------------------------------
def test_grid_basis_at_center(oracle):
    # test_grid.cpp:86-97
    b, start = oracle.basis(oracle.grid(3, 3), 0.0)
    np.testing.assert_allclose(b, [0, 1 / 48, 23 / 48, 23 / 48, 1 / 48, 0], atol=1e-12)
    assert start == 1
    np.testing.assert_array_equal(b, GOLD["basis_G3_at0"])


def test_partition_of_unity(oracle):
    # test_grid.cpp:115-131
    rng = np.random.default_rng(7)
    for G, P in [(3, 3), (5, 3), (3, 2), (8, 1)]:
        g = oracle.grid(G, P)
        for x in rng.uniform(-1, 1, 200):
            b, _ = oracle.basis(g, float(oracle.lib.kor_clamp(g, x)))
            assert abs(b.sum() - 1.0) < 1e-12


def test_quant_params_known_answers(oracle):
    # test_quant.cpp:12-42
    s, z, qh = oracle.quant_params(-1.0, 1.0, 8)
    assert abs(s - 2 / 255) < 1e-15 and z == 128 and qh == 255
    assert tuple(GOLD["qp_m1_1_8"]) == (s, z)
    s, z, _ = oracle.quant_params(0.0, 255.0, 8)
    assert s == 1.0 and z == 0
    s, z, _ = oracle.quant_params(-1.0, 1.0, 2)
    assert abs(s - 2 / 3) < 1e-15 and z == 2
    s, z, qh = oracle.quant_params(-1.0, 1.0, 8)
    assert oracle.lib.kor_quantize(0.5, s, z, 0, qh) == 192
    with pytest.raises(ValueError):
        oracle.quant_params(1.0, 1.0, 8)


def test_lut_table_known_answers(oracle):
    # test_lut.cpp:10-44
    assert len(oracle.lut(3, 1, 8)) == 5
    for p in (1, 2, 3):
        for k in (1, 4, 8):
            assert oracle.lut(p, k, 8)[0] == 0
    for k in (1, 2, 4, 8):
        for h in (3, 8):
            e = oracle.lut(3, k, h)
            s = 1.0 / ((1 << h) - 1)
            assert abs(e[-1] * s - 2.0 / 3.0) <= s
    with pytest.raises(ValueError):
        oracle.lut(3, 9, 8)
    with pytest.raises(ValueError):
        oracle.lut(3, 4, 1)


def test_lattice_aligns_with_knots(oracle):
    # test_quant.cpp:159-174: knot-aligned levels dequantize onto knots
    g = oracle.grid(3, 3)
    for k in (1, 4, 8):
        step = g.delta / (1 << k)
        for j in range(4):
            x = -1.0 + (j << k) * step
            assert oracle.level_of(g, k, x) == (j << k) or j == 3


def test_lookup_rejects_out_of_range(oracle):
    # test_lut.cpp:123-128
    g = oracle.grid(3, 3)
    lut = oracle.lut(3, 4, 8)
    with pytest.raises(IndexError):
        oracle.lut_lookup(g, 4, lut, -1)
    with pytest.raises(IndexError):
        oracle.lut_lookup(g, 4, lut, (3 << 4) + 1)


def test_all_ones_partition_bound(oracle):
    # test_lut.cpp:167-179
    g = oracle.grid(3, 3)
    ones = np.ones((6, 1))
    acts = (-1.0 + 2.0 * np.arange(32) / 31.0)[:, None]
    out = oracle.lut_forward(g, 4, 8, 32, acts, ones)
    slack = 6 * (1 / 255) / 2
    assert np.all(out >= 1 - slack) and np.all(out <= 1 + slack)


def test_im2col_padding_known_answer(oracle):
    # test_layers.cpp:122-139: padding fills borders with zeros
    x = np.array([[[1.0, 2.0], [3.0, 4.0]]])
    m = oracle.im2col(x, 3, 1, 1)
    assert m.shape == (4, 9)
    assert np.all(m.sum(1) == 10.0) and np.all((m == 0).sum(1) == 5)
    with pytest.raises(ValueError):
        oracle.im2col(np.zeros((1, 5, 5)), 2, 2, 0)


# ---- 3. against the reference compiled from /root/reference -----------------------
def test_exhaustive_lookup_equals_quantized_recursion(oracle, ref):
    # test_lut.cpp:54-81 / acceptance.cpp:223-257, widened to k=1..8, h=2..8
    n = 0
    for P in (1, 2, 3):
        for G in (1, 3, 5, 10):
            g = oracle.grid(G, P)
            for k in (1, 2, 3, 4, 8):
                for h in (2, 3, 8):
                    lut = oracle.lut(P, k, h)
                    L = G << k
                    for a in range(0, L + 1, max(1, L // 300)):
                        v1, s1 = oracle.lut_lookup(g, k, lut, a)
                        v2, s2 = ref.lut_lookup(G, P, k, h, a)
                        v3, s3 = oracle.quantized_basis_reference(g, k, h, a)
                        assert s1 == s2 == s3
                        np.testing.assert_array_equal(v1, v2)
                        np.testing.assert_array_equal(v1, v3)
                        n += len(v1)
    assert n > 10000


def test_levels_match_reference_random(oracle, ref):
    rng = np.random.default_rng(3)
    x = rng.uniform(-1.5, 1.5, 200000).astype(np.float32)
    for G, k in [(5, 8), (10, 8), (5, 2), (3, 3)]:
        np.testing.assert_array_equal(oracle.levels(oracle.grid(G, 3), k, x), ref.levels(G, 3, k, x))


def test_forwards_bit_exact_vs_reference(oracle, ref):
    rng = np.random.default_rng(11)
    for G in (3, 5, 10):
        nb = G + 3
        acts = rng.uniform(-1.2, 1.2, (40, 33))
        W = rng.normal(0, 0.1, (33 * nb, 9))
        g = oracle.grid(G, 3)
        np.testing.assert_array_equal(oracle.linear_forward(g, acts, W),
                                      ref.linear_forward(G, 3, acts, W))
        for k, h, bw in [(8, 8, 8), (4, 4, 4), (3, 3, 8), (2, 2, 2), (8, 8, 32)]:
            np.testing.assert_array_equal(oracle.lut_forward(g, k, h, bw, acts, W),
                                          ref.lut_forward(G, 3, k, h, bw, acts, W))


def test_integer_restatement_agrees_with_reference_lut_forward(oracle, ref):
    """acc - z_w*rowsum, scaled by s_b*s_w, equals tabulated_kan_forward to ~1e-11."""
    rng = np.random.default_rng(5)
    G, k, h = 5, 8, 8
    g = oracle.grid(G, 3)
    acts = rng.uniform(-1, 1, (64, 784)).astype(np.float32).astype(np.float64)
    W = rng.normal(0, 0.1, (784 * 8, 16))
    d = oracle.int_layer(g, k, h, 0, 8, W)
    lv = oracle.levels(g, k, acts.astype(np.float32))
    y = oracle.int_layer_forward(g, k, h, d, lv, 16)
    r = ref.lut_forward(G, 3, k, h, 8, acts, W)
    rel = np.abs(y - r).max() / np.abs(r).max()
    assert rel < 1e-10, rel


def test_conv_is_im2col_plus_linear(oracle, ref):
    # test_layers.cpp:149-176 through the reference itself
    rng = np.random.default_rng(31)
    x = rng.uniform(-1, 1, (3, 8, 8))
    W = rng.uniform(-1, 1, (3 * 9 * 6, 2))
    out = ref.conv_forward(3, 3, x, W, 2, 3, 1, 0)
    lin = oracle.linear_forward(oracle.grid(3, 3), oracle.im2col(x, 3, 1, 0), W)
    np.testing.assert_array_equal(out.reshape(2, -1).T, lin)


def test_reskan18_descriptor_is_rejected_by_reference(ref):
    text = open("/root/reference/proj/descriptors/reskan18.json").read() if os.path.exists(
        "/root/reference/proj/descriptors/reskan18.json") else None
    if text is None:
        pytest.skip("reference descriptors absent")
    with pytest.raises(ValueError, match="not positive integers"):
        ref.validate_descriptor(text)


# ---- conv path over lattice levels (implicit im2col) ------------------------------
@pytest.mark.parametrize("C,H,W,k,s,p", [(3, 8, 8, 3, 1, 1), (4, 9, 9, 3, 2, 1), (2, 7, 7, 1, 2, 0),
                                         (5, 6, 6, 3, 1, 0)])
def test_level_im2col_matches_reference_im2col(oracle, ref, C, H, W, k, s, p):
    """im2col over levels == levels of the reference's im2col (its zero padding
    becomes level(0.0)), in the reference's channel-major column order."""
    G, kk = 5, 8
    g = oracle.grid(G, 3)
    x = np.random.default_rng(C * H + k).uniform(-1, 1, (C, H, W))
    want = oracle.levels(g, kk, ref.im2col(x, k, s, p).astype(np.float32))
    lv = oracle.levels(g, kk, x.astype(np.float32))[None]
    got = oracle.im2col_levels(lv, k, s, p, oracle.level_of(g, kk, 0.0))
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("k,p", [(3, 1), (1, 0)])
def test_stride2_floor_recipe(oracle, ref, k, p):
    """floor-semantics stride 2 on 32x32 == the reference on the
    input zero-extended to 33x33, cropped to the top-left 16x16 outputs."""
    G, kk = 5, 8
    g = oracle.grid(G, 3)
    x = np.random.default_rng(k).uniform(-1, 1, (2, 32, 32))
    ext = np.zeros((2, 33, 33))
    ext[:, :32, :32] = x
    r = ref.im2col(ext, k, 2, p)  # [Ho*Wo, C*k*k] on the 33x33 input
    ho = (33 + 2 * p - k) // 2 + 1
    r = r.reshape(ho, ho, -1)[:16, :16].reshape(256, -1)
    lv = oracle.levels(g, kk, x.astype(np.float32))[None]
    got = oracle.im2col_levels(lv, k, 2, p, oracle.level_of(g, kk, 0.0))
    np.testing.assert_array_equal(got, oracle.levels(g, kk, r.astype(np.float32)))


def test_integer_conv_agrees_with_reference_conv(oracle, ref):
    """The oracle's integer conv (level im2col + integer layer, per-tensor u8 W)
    equals the reference's convkan_forward with LutBasis + fake-quant W to 1e-10."""
    G, k, h = 5, 8, 8
    rng = np.random.default_rng(8)
    x = rng.uniform(-1, 1, (2, 6, 8, 8)).astype(np.float32)
    W = rng.normal(0, 0.1, (6 * 9 * 8, 5))
    desc = {"grid": {"intervals": G, "degree": 3}, "input": [6, 8, 8],
            "layers": [{"type": "conv", "c_in": 6, "c_out": 5, "kernel": 3, "stride": 1,
                        "padding": 1}]}
    y = oracle.int_model_forward(desc, [W], [None], x.reshape(2, -1), k, h, 0, 8)
    for n in range(2):
        r = ref.conv_forward(G, 3, x[n].astype(np.float64), W, 5, 3, 1, 1, mode=1, k=k, h=h,
                             bits_w=8)
        assert np.abs(y[n] - r).max() / np.abs(r).max() < 1e-10


def test_extended_descriptor_validation():
    """Named tensors / residual / global_avgpool: shape errors surface like
    Model::validate's (ValueError through the C ABI)."""
    from paper_2603_17230_b200 import Engine, configs
    base = {"grid": {"intervals": 5, "degree": 3}, "input": [4, 8, 8]}
    bad = [
        [{"type": "conv", "c_in": 4, "c_out": 4, "kernel": 3, "padding": 1, "residual": "nope"}],
        [{"type": "conv", "c_in": 4, "c_out": 8, "kernel": 3, "padding": 1, "residual": "input"}],
        [{"type": "conv", "c_in": 4, "c_out": 4, "kernel": 3, "padding": 1, "id": "a"},
         {"type": "conv", "c_in": 4, "c_out": 4, "kernel": 3, "padding": 1, "id": "a"}],
        [{"type": "global_avgpool"}, {"type": "global_avgpool"}],
    ]
    for layers in bad:
        with pytest.raises(ValueError):
            Engine(dict(base, layers=layers), 0)
    # the ResKAN18 workload descriptor passes validation (only the device check fails here)
    try:
        Engine(configs.get("c5").descriptor(), 0)
    except RuntimeError:
        pass


def test_reference_composition_of_reskan_tracks_the_oracle(oracle, ref):
    """ResKAN blocks composed from reference functions (ref_graph_forward: LutBasis
    convs, fake-quant W, harness residual / pooling) agree with the oracle's
    integer restatement of the engine semantics (residual / pooled tensors
    carried as fp32 values, the rest as lattice levels) to 1e-9."""
    import json
    from paper_2603_17230_b200 import configs
    layers = configs.reskan18_layers(width=(8, 16), n_classes=10, in_ch=3)
    desc = {"name": "r", "grid": {"intervals": 5, "degree": 3}, "input": [3, 8, 8],
            "conv_output": "floor", "layers": layers}
    wl = configs.Workload("t", "t", [0], 5, 3, 1, 0.05, silu=False, input_shape=[3, 8, 8],
                          layers=layers)
    Ws, Bs = wl.weights()
    x = np.random.default_rng(0).uniform(-1, 1, (3, 192)).astype(np.float32)
    r = ref.graph_forward(json.dumps(desc), Ws, x.astype(np.float64), 10, k=8, h=8, threads=3)
    y = oracle.int_model_forward(desc, Ws, Bs, x, 8, 8, 0, 8)
    assert np.linalg.norm(y - r) / np.linalg.norm(r) < 1e-9

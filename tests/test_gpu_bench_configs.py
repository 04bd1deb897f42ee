"""Parity at the exact configurations bench.py measures (BASELINE.json configs,
through the C ABI), against the CPU oracle.

Every GPU forward here runs the FULL bench batch with the bench's own options
(configs.Workload.eval_options + bench.SPLIT_DEFAULT), so the engine makes the
same kernel, tile, table-variant, conv3 / gather and persistence choices the
bench does; the recorded launch plan (kan_engine_last_plan) is compared with
the committed one (tests/golden/bench_plans.json), which the bench line also
carries.  Rows of a batch are independent (no cross-sample op, layers.hpp:
99-211), so a spread of sampled rows is checked against the oracle:
  * integer LUT path: bit-exact (oracle int_model_forward: levels -> integer
    contraction -> fp64 epilogue -> next-layer levels / fp32 values),
  * bf16 path: 1e-2 norm-relative vs the host restatement of the bf16
    arithmetic (model) and vs the fp64 Cox-de Boor reference (per layer).
Reference: layers.hpp:99-190 (kan_linear_forward / convkan_forward),
eval.hpp:200-253 (model_forward), lut.hpp:44-47 / 217-231.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import bench  # noqa: E402
from paper_2603_17230_b200 import Engine, EvalOptions, OUT_I8, configs  # noqa: E402

PLANS = os.path.join(os.path.dirname(__file__), "golden", "bench_plans.json")
OUT_DIR = os.path.join(os.path.dirname(os.path.dirname(__file__)), "gpurun_out")


def bench_engine(wl, **over):
    Ws, Bs = wl.weights()
    e = Engine(wl.descriptor(), 0)
    for i, (w, b) in enumerate(zip(Ws, Bs)):
        e.set_coeffs(i, w, b)
    opts = EvalOptions(**wl.eval_options(), split_k=bench.per_config(bench.SPLIT_DEFAULT, wl.key, 0))
    for k, v in over.items():
        setattr(opts, k, v)
    e.configure(opts)
    e.set_option("record_plan", 1)
    return e, Ws, Bs, opts


def check_plan(key, plan):
    """The forward's launch plan equals the committed bench plan (written to
    gpurun_out/ for review when no plan is committed yet)."""
    lines = plan.strip().splitlines()
    assert lines, "empty launch plan"
    os.makedirs(OUT_DIR, exist_ok=True)
    with open(os.path.join(OUT_DIR, f"plan_{key}.txt"), "w") as f:
        f.write(plan)
    if os.path.exists(PLANS):
        with open(PLANS) as f:
            want = json.load(f)
        if key in want:
            assert lines == want[key], f"{key}: launch plan differs from tests/golden/bench_plans.json"


def sample_rows(n, count, seed):
    rng = np.random.default_rng(seed)
    mid = rng.choice(np.arange(1, n - 1), count - 2, replace=False)
    return np.sort(np.concatenate([[0, n - 1], mid]))


@pytest.mark.parametrize("key", ["c5", "c5pc"])
def test_c5_full_reskan18_bit_exact(oracle, key):
    """Full ResKAN18 (64/128/256/512 channels, 3x32x32, k8/h3) at batch 8192:
    16 sampled images' logits bit-exact with the oracle.  c5 = the reference
    weight scheme (the bench headline), c5pc = per-channel int8 + SiLU."""
    wl = configs.get(key)
    B = wl.batch
    x = wl.inputs(B, seed=100)  # the bench's first resident batch
    e, Ws, Bs, _ = bench_engine(wl)
    y = e.model_forward(torch.from_numpy(x).cuda()).cpu().numpy()
    check_plan(key, e.last_plan)
    assert np.isfinite(y).all()
    rows = sample_rows(B, 16, 5)
    yo = oracle.int_model_forward(wl.descriptor(), Ws, Bs, x[rows], wl.lut_k, wl.lut_h, wl.wscheme, wl.bits_w)
    np.testing.assert_array_equal(y[rows], yo.astype(np.float32))


def test_c3_full_mlp_bit_exact(oracle):
    """C3 [3072,1024,1024,10], G=10, k8/h8 int8 + SiLU at batch 65,536 (bench
    options): 64 sampled rows bit-exact, hidden levels included implicitly
    (the logits depend on every hidden level)."""
    wl = configs.get("c3")
    B = wl.batch
    x = wl.inputs(B, seed=100)
    e, Ws, Bs, _ = bench_engine(wl)
    y = e.model_forward(torch.from_numpy(x).cuda()).cpu().numpy()
    check_plan("c3", e.last_plan)
    rows = sample_rows(B, 64, 6)
    yo = oracle.int_model_forward(wl.descriptor(), Ws, Bs, x[rows], wl.lut_k, wl.lut_h, wl.wscheme, wl.bits_w)
    np.testing.assert_array_equal(y[rows], yo.astype(np.float32))


def float_reference(oracle, wl, Ws, Bs, x):
    """fp64 restatement of the float paths: Cox-de Boor basis (grid.hpp:124-182)
    contracted with W (layers.hpp:99-121) plus silu(clamp_to_domain(x)) . W_b,
    layer by layer with no inter-layer activation (eval.hpp:135-193)."""
    g = oracle.grid(wl.G, wl.P)
    h = x.astype(np.float64)
    hi_open = np.nextafter(1.0, -1.0)
    for w, b in zip(Ws, Bs):
        y = oracle.linear_forward(g, h, w)
        if b is not None:
            c = np.clip(h, -1.0, hi_open)
            y = y + (c / (1.0 + np.exp(-c))) @ b
        h = y
    return h


def bf16_round(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).to(torch.float32).numpy()


def bf16_restatement(oracle, wl, Ws, Bs, x):
    """The bf16 path's arithmetic restated on the host: each layer's basis
    values (fp64 Cox-de Boor of the clamped input) and SiLU values rounded to
    bf16, weights rounded to bf16, products summed in fp64, the layer output
    rounded to the fp32 the engine stores between layers."""
    G, P = wl.G, wl.P
    nb = G + P
    g = oracle.grid(G, P)
    h = x.astype(np.float32)
    for w, b in zip(Ws, Bs):
        M, n_in = h.shape
        B = np.zeros((M, n_in * nb))
        hc = np.clip(h.astype(np.float64), -1.0, np.nextafter(1.0, -1.0))  # clamp_to_domain
        for m in range(M):
            for i in range(n_in):
                B[m, i * nb:(i + 1) * nb] = oracle.basis(g, float(hc[m, i]))[0]
        y = bf16_round(B).astype(np.float64) @ bf16_round(w).astype(np.float64)
        if b is not None:
            c = np.clip(h.astype(np.float64), -1.0, np.nextafter(1.0, -1.0))
            y += bf16_round(c / (1.0 + np.exp(-c))).astype(np.float64) @ bf16_round(b).astype(np.float64)
        h = y.astype(np.float32)
    return h.astype(np.float64)


def test_c3_bf16_full_mlp(oracle):
    """C3 bf16 path at batch 65,536 (bench options): 16 sampled rows within
    1e-2 (norm-relative) of the host restatement of the bf16 arithmetic, and
    each layer on its own within 1e-2 of the fp64 Cox-de Boor reference (the
    north_star bar).  Through three layers the bf16 operand rounding itself
    moves the logits by several percent against fp64 (printed), so the model
    bar is against the bf16 restatement."""
    wl = configs.get("c3bf16")
    B = wl.batch
    x = wl.inputs(B, seed=100)
    e, Ws, Bs, _ = bench_engine(wl)
    y = e.model_forward(torch.from_numpy(x).cuda()).cpu().numpy()
    check_plan("c3bf16", e.last_plan)
    rows = sample_rows(B, 16, 7)
    emu = bf16_restatement(oracle, wl, Ws, Bs, x[rows])
    err = float(np.linalg.norm(y[rows] - emu) / np.linalg.norm(emu))
    r64 = float_reference(oracle, wl, Ws, Bs, x[rows])
    print(f"C3 bf16: vs bf16 restatement {err:.2e}, vs fp64 {np.linalg.norm(y[rows] - r64) / np.linalg.norm(r64):.2e}")
    assert err < 1e-2, err
    # per layer against fp64: layer li alone, fed fp32 inputs in [-1.1, 1.1]
    dims = wl.dims
    for li in range(len(Ws)):
        lw = configs.Workload("l", "l", [dims[li], dims[li + 1]], wl.G, wl.P, 4096, wl.std, mode="bf16")
        el = Engine(lw.descriptor(), 0)
        el.set_coeffs(0, Ws[li], Bs[li])
        el.configure(EvalOptions(mode="bf16", silu_base=True))
        xl = np.random.default_rng(li).uniform(-1.1, 1.1, (4096, dims[li])).astype(np.float32)
        yl = el.model_forward(torch.from_numpy(xl).cuda()).cpu().numpy()
        rl = float_reference(oracle, lw, [Ws[li]], [Bs[li]], xl[:64])
        el_err = float(np.linalg.norm(yl[:64] - rl) / np.linalg.norm(rl))
        assert el_err < 1e-2, (li, el_err)


@pytest.mark.parametrize("key", ["c1", "c2"])
def test_c1_c2_bench_path_bit_exact(oracle, key):
    """C1/C2 with the bench's split (unsplit persistent launches, the output
    layer as its own launch) and output kind (C2: int8 logits at the bench's
    calibrated scale): every row bit-exact, hidden levels through the logits."""
    wl = configs.get(key)
    B = wl.batch
    x = wl.inputs(B, seed=100)
    e, Ws, Bs, opts = bench_engine(wl)
    xd = torch.from_numpy(x).cuda()
    if wl.int8_out:
        yf = e.model_forward(xd).float()
        opts.out_kind, opts.out_scale = OUT_I8, float(yf.abs().max().item()) / 127.0
        e.configure(opts)
    y = e.model_forward(xd).cpu().numpy()
    check_plan(key, e.last_plan)
    yo = oracle.int_model_forward(wl.descriptor(), Ws, Bs, x, wl.lut_k, wl.lut_h, wl.wscheme, wl.bits_w)
    if wl.int8_out:
        yo = np.array([[oracle.requant_i8(v, opts.out_scale) for v in row] for row in yo], np.int8)
        np.testing.assert_array_equal(y, yo)
    else:
        np.testing.assert_array_equal(y, yo.astype(np.float32))


def test_c4_full_conv_bit_exact(oracle):
    """C4 KAN conv 3x3 64->64 on 32x32 at batch 256 (bench options): 16 sampled
    images bit-exact."""
    wl = configs.get("c4")
    B = wl.batch
    x = wl.inputs(B, seed=100)
    e, Ws, Bs, _ = bench_engine(wl)
    y = e.model_forward(torch.from_numpy(x).cuda()).cpu().numpy()
    check_plan("c4", e.last_plan)
    rows = sample_rows(B, 16, 8)
    yo = oracle.int_model_forward(wl.descriptor(), Ws, Bs, x[rows], wl.lut_k, wl.lut_h, wl.wscheme, wl.bits_w)
    np.testing.assert_array_equal(y[rows], yo.astype(np.float32).reshape(len(rows), -1))

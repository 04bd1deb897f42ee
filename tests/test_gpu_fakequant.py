"""GPU fake-quant mode (EvalMode::kFakeQuant, eval.hpp:106-159) and the GPU
sweep backend (evaluate_accuracy, run_sweep) against the oracle restatement
(pinned to the reference in tests/test_oracle_pins.py) and the reference's
own model_forward.  Fake-quant runs exact fp64 per-connection tables rounded
once to fp32 and summed in fp32: bar ||y - ref|| / ||ref|| < 1e-4."""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2603_17230_b200 import Engine, EvalOptions  # noqa: E402
from paper_2603_17230_b200.sweep import SweepSpec, run_sweep  # noqa: E402

TOL = 1e-4
MLP = {"name": "m", "grid": {"intervals": 5, "degree": 3}, "input": [64],
       "layers": [{"type": "linear", "n_in": 64, "n_out": 32}, {"type": "linear", "n_in": 32, "n_out": 10}]}
LEKAN = {"name": "LeKAN", "grid": {"intervals": 3, "degree": 3}, "input": [1, 28, 28],
         "layers": [{"type": "conv", "c_in": 1, "c_out": 6, "kernel": 5, "stride": 1, "padding": 0},
                    {"type": "maxpool", "window": 2},
                    {"type": "conv", "c_in": 6, "c_out": 16, "kernel": 5, "stride": 1, "padding": 2},
                    {"type": "maxpool", "window": 2}, {"type": "flatten"},
                    {"type": "linear", "n_in": 576, "n_out": 10}]}


def _ws(desc, seed, std=0.1):
    rng = np.random.default_rng(seed)
    nb = desc["grid"]["intervals"] + desc["grid"]["degree"]
    out = []
    for l in desc["layers"]:
        if l["type"] == "linear":
            out.append(rng.normal(0, std, (l["n_in"] * nb, l["n_out"])))
        elif l["type"] == "conv":
            out.append(rng.normal(0, std, (l["c_in"] * l["kernel"] ** 2 * nb, l["c_out"])))
    return out


def _engine(desc, ws):
    e = Engine(desc, 0)
    for i, w in enumerate(ws):
        e.set_coeffs(i, w)
    return e


def _rel(y, r):
    return np.linalg.norm(y - r) / max(np.linalg.norm(r), 1e-30)


@pytest.mark.parametrize("bw,ba,bb", [(8, 8, 8), (4, 6, 3), (32, 8, 32), (3, 2, 2), (8, 5, 32), (32, 32, 32),
                                      (6, 32, 32)])
def test_fake_quant_mlp(oracle, ref, bw, ba, bb):
    ws = _ws(MLP, ba * 10 + bb)
    e = _engine(MLP, ws)
    e.configure(EvalOptions(mode="fake-quant", bits_w=bw, lut_k=ba, lut_h=bb))
    x = np.random.default_rng(1).uniform(-1.2, 1.2, (500, 64)).astype(np.float32)
    y = e.model_forward(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
    want = oracle.fakequant_model_forward(MLP, ws, x.astype(np.float64), bw, ba, bb)
    assert _rel(y, want) < TOL
    r = ref.model_forward(json.dumps(MLP), ws, x.astype(np.float64), 10, mode=1, k=ba, h=bb, bits_w=bw)
    assert _rel(y, r) < TOL


def test_fake_quant_conv_model(oracle):
    ws = _ws(LEKAN, 3)
    e = _engine(LEKAN, ws)
    x = np.random.default_rng(2).uniform(-1, 1, (16, 784)).astype(np.float32)
    for bw, ba, bb in ((8, 8, 8), (5, 4, 6)):
        e.configure(EvalOptions(mode="fake-quant", bits_w=bw, lut_k=ba, lut_h=bb))
        y = e.model_forward(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
        want = oracle.fakequant_model_forward(LEKAN, ws, x.astype(np.float64), bw, ba, bb)
        assert _rel(y, want) < TOL


def test_fake_quant_unsupported_combination_fails_loudly():
    e = _engine(MLP, _ws(MLP, 0))
    with pytest.raises(NotImplementedError):
        e.configure(EvalOptions(mode="fake-quant", bits_w=8, lut_k=32, lut_h=4))


def test_sweep_matches_reference_accuracy(ref):
    """run_sweep over all three modes: the GPU accuracies agree with the
    reference's predict on the same rows (labels = the fp32 model's argmax,
    so accuracies are informative)."""
    ws = _ws(MLP, 11)
    e = _engine(MLP, ws)
    x = np.random.default_rng(5).uniform(-1, 1, (2000, 64)).astype(np.float32)
    text = json.dumps(MLP)
    labels = ref.model_forward(text, ws, x.astype(np.float64), 10, mode=0).argmax(1).astype(np.int32)
    spec = SweepSpec([8, 4], [8, 4, 3], [8, 3], ["fake-quant", "bspline-lut", "spline-table"])
    xd, ld = torch.from_numpy(x).cuda(), torch.from_numpy(labels).cuda()
    points, pb, pm = run_sweep(e, xd, ld, spec, MLP)
    assert len(points) == 12 + 12 + 6 and pb and pm
    for p in points:
        c = p.config
        mode = {"fake-quant": 1, "bspline-lut": 2, "spline-table": 3}[c.mode]
        r = ref.model_forward(text, ws, x.astype(np.float64), 10, mode=mode, k=c.bits_a, h=c.bits_b,
                              bits_w=c.bits_w if c.bits_w != 32 else 8)
        want = float((r.argmax(1) == labels).mean())
        if c.mode == "spline-table":
            assert p.accuracy == want, (c, p.accuracy, want)  # bit-exact path
        else:
            assert abs(p.accuracy - want) <= 0.005, (c, p.accuracy, want)


@pytest.mark.parametrize("desc", [MLP, LEKAN])
def test_fake_quant_calibrated_ranges(ref, desc):
    """QuantConfig::ARangePolicy::kCalibrated: per-layer activation quantizers
    from the reference's calibrate_activation_ranges (eval.hpp:289-341)."""
    ws = _ws(desc, 7)
    e = _engine(desc, ws)
    D = int(np.prod(desc["input"]))
    rng = np.random.default_rng(3)
    calib = rng.uniform(-1, 1, (64, D))
    x = rng.uniform(-1, 1, (200 if D < 100 else 12, D)).astype(np.float32)
    text = json.dumps(desc)
    nk = sum(l["type"] in ("linear", "conv") for l in desc["layers"])
    ranges = ref.calibrate_ranges(text, ws, calib, nk)
    for bw, ba, bb in ((8, 8, 8), (6, 5, 4)):
        e.configure(EvalOptions(mode="fake-quant", bits_w=bw, lut_k=ba, lut_h=bb, a_ranges=ranges))
        y = e.model_forward(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
        r = ref.fakequant_calibrated_forward(text, ws, x.astype(np.float64), 10, bw, ba, bb, ranges)
        assert _rel(y, r) < TOL
    with pytest.raises(ValueError):
        e.configure(EvalOptions(mode="fake-quant", bits_w=8, lut_k=8, lut_h=8, a_ranges=ranges[:1]))

"""Small forwards of every kernel family, for compute-sanitizer (racecheck,
memcheck, synccheck; one tool per run):

    python scripts/sanitize_small.py            # plain run first (must exit 0)
    compute-sanitizer --tool racecheck python scripts/sanitize_small.py

Covers: gather GEMM (persistent and split-K, fused output layer, int8 logits),
small-N layer, kan_conv3 (SiLU, per-channel), kan_convw (zero point,
per-channel and SiLU forms, 8/16/32 images per tile, ky-merged and per-tap
issue, lockstep rings), the general conv kernel, level
prepass, stem im2col, pooling, spline-table and fp32 paths.  Results are
checked against each other (bit-identical across kernel choices) so a run
that races also fails here.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2603_17230_b200 import Engine, EvalOptions, OUT_I8, configs  # noqa: E402


def build(desc, Ws, Bs, options=None, **opts):
    e = Engine(desc, 0)
    for i, (w, b) in enumerate(zip(Ws, Bs)):
        e.set_coeffs(i, w, b)
    for k, v in (options or {}).items():
        e.set_option(k, v)
    e.configure(EvalOptions(**opts))
    return e


def run(e, x):
    y = e.model_forward(torch.from_numpy(x).cuda()).cpu().numpy()
    torch.cuda.synchronize()
    return y


def main():
    # MLP: persistent vs split-K (fused output layer) vs int8 logits
    wl = configs.Workload("m", "m", [200, 64, 10], 5, 3, 1, 0.1)
    Ws, Bs = wl.weights()
    x = wl.inputs(300, seed=1)
    desc = wl.descriptor()
    base = dict(mode="bspline-lut", lut_k=8, lut_h=8, bits_w=8, w_scheme=1, silu_base=True)
    Wm, Bm, xm = Ws, Bs, x
    y1 = run(build(desc, Ws, Bs, split_k=1, **base), x)
    y2 = run(build(desc, Ws, Bs, split_k=2, **base), x)
    assert np.array_equal(y1, y2), "MLP split-K differs"
    e = build(desc, Ws, Bs, out_kind=OUT_I8, out_scale=0.05, **base)
    run(e, x)
    run(build(desc, Ws, Bs, options={"level_prepass_min": 0}, **base), x)
    run(build(desc, Ws, Bs, mode="fp32", silu_base=True), x)
    run(build(desc, Ws, [None, None], mode="spline-table", lut_k=4, lut_h=4), x)

    # ResKAN (4 stages: 32/16/8/4-wide maps), both weight schemes, batch 19
    layers = configs.reskan18_layers(width=(8, 16, 32, 64), n_classes=10, in_ch=3)
    for ws in (0, 1):
        rw = configs.Workload("r", "r", [0], 5, 3, 1, 0.05, silu=False, wscheme=ws, lut_h=3,
                              input_shape=[3, 32, 32], layers=layers,
                              extra={"descriptor": {"conv_output": "floor"}})
        Ws, Bs = rw.weights()
        x = rw.inputs(19, seed=2)
        o = rw.eval_options()
        ya = run(build(rw.descriptor(), Ws, Bs, **o), x)
        yb = run(build(rw.descriptor(), Ws, Bs, options={"no_convw": 1}, **o), x)
        assert np.array_equal(ya, yb), f"convw vs gather differ (scheme {ws})"
    # kan_conv3 with the SiLU term (per-channel), C4-like shape at small batch
    cw = configs.Workload("c", "c", [0], 5, 3, 1, 0.05, input_shape=[32, 32, 32],
                          layers=[{"type": "conv", "c_in": 32, "c_out": 32, "kernel": 3, "stride": 1, "padding": 1},
                                  {"type": "conv", "c_in": 32, "c_out": 32, "kernel": 3, "stride": 1, "padding": 1},
                                  {"type": "maxpool", "window": 2}, {"type": "flatten"},
                                  {"type": "linear", "n_in": 32 * 16 * 16, "n_out": 10}])
    Ws, Bs = cw.weights()
    x = cw.inputs(20, seed=3)  # >= 148 tiles: kan_conv3 takes the 3x3 layers
    o = dict(mode="bspline-lut", lut_k=8, lut_h=8, bits_w=8, w_scheme=1, silu_base=True)
    ya = run(build(cw.descriptor(), Ws, Bs, **o), x)  # kan_convw, SiLU form
    yc = run(build(cw.descriptor(), Ws, Bs, options={"no_convw": 1}, **o), x)  # kan_conv3
    yb = run(build(cw.descriptor(), Ws, Bs, options={"no_convw": 1, "no_conv3": 1}, **o), x)  # gather GEMM
    assert np.array_equal(ya, yb), "convw (SiLU) vs gather differ"
    assert np.array_equal(yc, yb), "conv3 vs gather differ"
    yl = run(build(cw.descriptor(), Ws, Bs, options={"convw_lock": 1}, **o), x)
    yk = run(build(cw.descriptor(), Ws, Bs, options={"convw_no_kym": 1}, **o), x)
    assert np.array_equal(ya, yl) and np.array_equal(ya, yk), "convw issue variants differ"
    # persistent launch with the fused output layer (opt-in) vs its own launch
    yp = run(build(desc, Wm, Bm, options={"fuse_persistent": 1}, split_k=1, **base), xm)
    assert np.array_equal(yp, y1), "persistent fused output layer differs"
    print("sanitize_small: ok")


if __name__ == "__main__":
    main()

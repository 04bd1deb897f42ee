"""Probe single conv configurations (debug aid): python scripts/conv_probe.py C H W co k s p"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_17230_b200 import Engine, EvalOptions, W_PER_CHANNEL_SYM, configs
from oracle.pyoracle import Oracle
C, H, W, co, k, s, p = map(int, sys.argv[1:8])
mode = sys.argv[8] if len(sys.argv) > 8 else "bspline-lut"
split = int(sys.argv[9]) if len(sys.argv) > 9 else 0
desc = {"name": "c", "grid": {"intervals": 5, "degree": 3}, "input": [C, H, W], "conv_output": "floor",
        "layers": [{"type": "conv", "c_in": C, "c_out": co, "kernel": k, "stride": s, "padding": p}]}
wl = configs.Workload("t", "t", [0], 5, 3, 1, 0.05, input_shape=desc["input"], layers=desc["layers"])
Ws, Bs = wl.weights()
e = Engine(desc, 0)
e.set_coeffs(0, Ws[0], Bs[0])
e.configure(EvalOptions(mode=mode, lut_k=8, lut_h=8, bits_w=8, w_scheme=W_PER_CHANNEL_SYM, silu_base=True, split_k=split))
x = np.random.default_rng(0).uniform(-1, 1, (2, C * H * W)).astype(np.float32)
y = e.model_forward(torch.from_numpy(x).cuda()).cpu().numpy()
if mode == "bspline-lut":
    yo = Oracle().int_model_forward(desc, Ws, Bs, x, 8, 8, W_PER_CHANNEL_SYM, 8).astype(np.float32).reshape(2, -1)
    print("OK" if np.array_equal(y, yo) else f"MISMATCH {np.mean(y != yo):.4f}")
else:
    print("ran")

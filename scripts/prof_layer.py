"""Run a workload's forward a few times without CUDA graphs (for ncu captures).

    python scripts/prof_layer.py [--config c2] [--iters 6] [--batch N]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2603_17230_b200 import Engine, EvalOptions, W_PER_CHANNEL_SYM  # noqa: E402
from paper_2603_17230_b200 import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--split", type=int, default=0)
    a = ap.parse_args()
    wl = configs.get(a.config)
    B = a.batch or wl.batch
    Ws, Bs = wl.weights()
    e = Engine(wl.descriptor(), 0)
    for i, (w, b) in enumerate(zip(Ws, Bs)):
        e.set_coeffs(i, w, b)
    e.configure(EvalOptions(mode=wl.mode, lut_k=wl.lut_k, lut_h=wl.lut_h, bits_w=wl.bits_w,
                            w_scheme=W_PER_CHANNEL_SYM, silu_base=wl.silu, split_k=a.split))
    x = torch.from_numpy(wl.inputs(B)).cuda()
    e.set_profiling(True)
    for _ in range(a.iters):
        e.model_forward(x)
    torch.cuda.synchronize()
    for li in range(len(wl.dims) - 1):
        ms, n = e.layer_time_ms(li)
        print(f"layer {li}: {ms / max(n, 1) * 1e3:.1f} us avg over {n}")


if __name__ == "__main__":
    main()

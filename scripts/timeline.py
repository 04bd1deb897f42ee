"""Per-CTA phase breakdown of each layer's gather-GEMM launch (engine option timeline=1).

    python scripts/timeline.py --config c2 [--split S] [--batch B]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_17230_b200 import Engine, EvalOptions, W_PER_CHANNEL_SYM  # noqa: E402
from paper_2603_17230_b200 import configs  # noqa: E402

NAMES = ["start", "tables", "stage0", "lastA", "tmemfull", "partials", "done", "reduced"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--split", type=int, default=0)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--mode", default="")
    a = ap.parse_args()
    wl = configs.get(a.config)
    B = a.batch or wl.batch
    Ws, Bs = wl.weights()
    e = Engine(wl.descriptor(), 0)
    e.set_option("timeline", 1)
    for i, (w, b) in enumerate(zip(Ws, Bs)):
        e.set_coeffs(i, w, b)
    e.configure(EvalOptions(mode=a.mode or wl.mode, lut_k=wl.lut_k, lut_h=wl.lut_h,
                            bits_w=wl.bits_w, w_scheme=W_PER_CHANNEL_SYM, silu_base=wl.silu,
                            split_k=a.split))
    x = torch.from_numpy(wl.inputs(B)).cuda()
    for _ in range(3):
        e.model_forward(x)
    torch.cuda.synchronize()
    for li in range(wl.n_kan):
        t = e.layer_timeline(li).astype(np.int64)
        if t.size == 0:
            continue
        t0 = t[:, 0].min()
        rel = (t - t0) / 1e3  # us
        rel[t == 0] = np.nan
        print(f"layer {li}: {t.shape[0]} CTAs, kernel span {np.nanmax(rel):.1f} us")
        for k, n in enumerate(NAMES):
            col = rel[:, k]
            if np.all(np.isnan(col)):
                continue
            print(f"   {n:9s} min {np.nanmin(col):8.2f}  med {np.nanmedian(col):8.2f}  max {np.nanmax(col):8.2f}")
        d = rel[:, 3] - rel[:, 2]
        print(f"   mainloop (stage0->lastA) med {np.nanmedian(d):.2f} us")
        own = rel - rel[:, :1]  # each CTA relative to its own start
        print("   per-CTA (from own start) medians: " + ", ".join(
            f"{n} {np.nanmedian(own[:, k]):.2f}" for k, n in enumerate(NAMES)
            if not np.all(np.isnan(own[:, k]))))


if __name__ == "__main__":
    main()

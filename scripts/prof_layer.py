"""Per-layer device time of a workload's forward, replayed from a CUDA graph so
host launch gaps stay out of the CUDA-event brackets (also used under ncu).

    python scripts/prof_layer.py [--config c2] [--iters 20] [--batch N] [--split S] [--nograph]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2603_17230_b200 import Engine, EvalOptions  # noqa: E402
from paper_2603_17230_b200 import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--split", type=int, default=0)
    ap.add_argument("--nograph", action="store_true")
    ap.add_argument("--mode", default="")
    ap.add_argument("--opt", action="append", default=[], help="engine option name=value (repeatable)")
    a = ap.parse_args()
    wl = configs.get(a.config)
    B = a.batch or wl.batch
    Ws, Bs = wl.weights()
    e = Engine(wl.descriptor(), 0)
    for i, (w, b) in enumerate(zip(Ws, Bs)):
        e.set_coeffs(i, w, b)
    for kv in a.opt:
        k, v = kv.split("=")
        e.set_option(k, int(v))
    o = wl.eval_options()
    if a.mode:
        o["mode"] = a.mode
    e.configure(EvalOptions(**o, split_k=a.split))
    x = torch.from_numpy(wl.inputs(B)).cuda()
    out = e.model_forward(x)  # warm-up: allocations, lazy module load
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    if a.nograph:
        e.set_profiling(True)
        with torch.cuda.stream(st):
            for _ in range(a.iters):
                e.model_forward(x, out=out, stream=st)
    else:
        e.set_profiling(True)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(a.iters):
                e.model_forward(x, out=out, stream=st)
        g.replay()
    torch.cuda.synchronize()
    for li in range(wl.n_kan):
        ms, n = e.layer_time_ms(li)
        print(f"layer {li}: {ms / max(n, 1) * 1e3:.2f} us avg over {n}")


if __name__ == "__main__":
    main()

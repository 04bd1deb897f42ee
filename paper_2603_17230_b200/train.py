"""GPU training of KAN MLPs, mirroring the reference's train() for linear
stacks (train.hpp:162-410): minibatch SGD with momentum on softmax
cross-entropy.

Forward: each layer is its own fp32 engine (the Cox-de Boor datapath), so the
layer inputs the backward needs stay on the device.  Backward:
kan_engine_linear_backward per layer (d_coeffs, d_inputs; the bottom layer
skips d_inputs, train.hpp:358), softmax_cross_entropy on the GPU.  Update
(train.hpp:361-366): v = momentum * v - lr * g; w += v, applied in fp64 on
the host copy and pushed back with set_coeffs (one upload per layer per step).
Conv layers (train.hpp:367-400, col2im) are not covered.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from .engine import Engine, EvalOptions, softmax_cross_entropy


@dataclass
class TrainConfig:
    lr: float = 1e-3
    momentum: float = 0.9
    epochs: int = 10
    batch: int = 64
    seed: int = 0


class MlpTrainer:
    def __init__(self, descriptor: dict, coeffs: List[np.ndarray], cfg: TrainConfig, device: int = 0):
        if any(l["type"] != "linear" for l in descriptor["layers"]):
            raise NotImplementedError("MlpTrainer trains linear KAN stacks (no conv / pooling)")
        self.cfg = cfg
        self.desc = descriptor
        self.coeffs = [np.array(c, dtype=np.float64) for c in coeffs]
        self.vel = [np.zeros_like(c) for c in self.coeffs]
        g = descriptor["grid"]
        self.engines = []
        for l, c in zip(descriptor["layers"], self.coeffs):
            d = {"name": "layer", "grid": g, "input": [l["n_in"]], "layers": [l]}
            if "domain" in descriptor:
                d["domain"] = descriptor["domain"]
            e = Engine(d, device)
            e.set_coeffs(0, c)
            e.configure(EvalOptions(mode="fp32"))
            self.engines.append(e)

    def forward(self, x):
        acts = [x]
        for e in self.engines:
            acts.append(e.model_forward(acts[-1]))
        return acts

    def step(self, x, labels) -> float:
        """One minibatch: forward, loss, backward, momentum update; returns the loss."""
        acts = self.forward(x)
        loss, d = softmax_cross_entropy(acts[-1], labels)
        for li in range(len(self.engines) - 1, -1, -1):
            dc, di = self.engines[li].linear_backward(0, acts[li], d, want_inputs=li > 0)
            g = dc.double().cpu().numpy()
            self.vel[li] = self.cfg.momentum * self.vel[li] - self.cfg.lr * g
            self.coeffs[li] += self.vel[li]
            d = di
        for e, c in zip(self.engines, self.coeffs):
            e.set_coeffs(0, c)
            e.configure(EvalOptions(mode="fp32"))
        return loss

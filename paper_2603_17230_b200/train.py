"""GPU training of KAN models, mirroring the reference's train()
(train.hpp:162-462): minibatch SGD with momentum on softmax cross-entropy,
over the reference layer set (linear, conv, maxpool, flatten).

Forward: each KAN layer is its own fp32 engine (the Cox-de Boor datapath; conv
layers through fp32 im2col rows), maxpool2 a GPU kernel, flatten a view; the
layer inputs the backward needs stay on the device.  Backward, last layer
first: kan_engine_linear_backward / kan_engine_conv_backward (d_coeffs,
d_inputs; the bottom layer skips d_inputs, train.hpp:358, 392), the pooling
backward (train.hpp:407-431), softmax_cross_entropy on the GPU.  Update
(train.hpp:361-366, 401-404): v = momentum * v - lr * g; w += v, on the device
(kan_engine_sgd_step: fp64 master coefficients and velocity stay resident, the
fp32 working copies are refreshed in the same launch; nothing crosses PCIe in
a step except the loss).  `coeffs` reads the current coefficients back.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np

from . import configs as _configs
from .engine import Engine, EvalOptions, maxpool2, maxpool2_backward, softmax_cross_entropy


@dataclass
class TrainConfig:
    lr: float = 1e-3
    momentum: float = 0.9
    epochs: int = 10
    batch: int = 64
    seed: int = 0


class Trainer:
    def __init__(self, descriptor: dict, coeffs: List[np.ndarray], cfg: TrainConfig, device: int = 0):
        for l in descriptor["layers"]:
            if l["type"] not in ("linear", "conv", "maxpool", "flatten") or \
                    {"id", "input_from", "residual"} & set(l):
                raise NotImplementedError("train() covers the reference layer set (linear, conv, maxpool, flatten)")
        self.cfg = cfg
        self.desc = descriptor
        self.shapes = _configs.walk_shapes(descriptor)
        init = [np.array(c, dtype=np.float64) for c in coeffs]
        self.engines = []  # per layer: an fp32 single-layer engine, or None
        ki = 0
        for s in self.shapes:
            if s["type"] in ("linear", "conv"):
                d = {"name": "layer", "grid": descriptor["grid"], "input": list(s["in"]), "layers": [s["layer"]]}
                if "domain" in descriptor:
                    d["domain"] = descriptor["domain"]
                e = Engine(d, device)
                e.set_coeffs(0, init[ki])
                e.configure(EvalOptions(mode="fp32"))
                self.engines.append(e)
                ki += 1
            else:
                self.engines.append(None)

    @property
    def coeffs(self) -> List[np.ndarray]:
        """Current coefficients of every KAN layer (read back from the device)."""
        return [e.get_coeffs(0) for e in self.engines if e is not None]

    def forward(self, x):
        """Per-layer inputs and the logits (rows [batch, values])."""
        acts = [x]
        for s, e in zip(self.shapes, self.engines):
            cur = acts[-1]
            if s["type"] in ("linear", "conv"):
                acts.append(e.model_forward(cur.contiguous()))
            elif s["type"] == "maxpool":
                c, h, w = s["in"]
                acts.append(maxpool2(cur, c, h, w, s["layer"].get("window", 2)))
            else:  # flatten: NCHW rows are already the reference's flat order
                acts.append(cur)
        return acts

    def step(self, x, labels) -> float:
        """One minibatch: forward, loss, backward, momentum update; returns the loss."""
        acts = self.forward(x)
        loss, d = softmax_cross_entropy(acts[-1], labels)
        ki = sum(1 for e in self.engines if e is not None)
        for li in range(len(self.shapes) - 1, -1, -1):
            s, e = self.shapes[li], self.engines[li]
            want = li > 0
            if s["type"] == "linear":
                ki -= 1
                dc, d = e.linear_backward(0, acts[li], d, want_inputs=want)
            elif s["type"] == "conv":
                ki -= 1
                dc, d = e.conv_backward(0, acts[li], d, want_inputs=want)
            elif s["type"] == "maxpool":
                c, h, w = s["in"]
                d = maxpool2_backward(acts[li], d, c, h, w, s["layer"].get("window", 2))
                continue
            else:
                continue
            e.sgd_step(0, dc, self.cfg.lr, self.cfg.momentum)
        return loss


MlpTrainer = Trainer  # the linear-stack case

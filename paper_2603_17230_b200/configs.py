"""The five BASELINE.json workloads, as descriptors + seeded synthetic data.

Descriptors use the reference's JSON schema (io.hpp:357-386).  Data is
synthetic with the shapes and distributions BASELINE.json states (MNIST /
CIFAR are not available and are not used):
  inputs  ~ U[-1, 1] fp32
  spline coefficients ~ N(0, std) (0.1 for C1/C2, 0.05 for C3-C5)
  base (SiLU) weights  ~ N(0, 1/sqrt(n_in))
Algorithmic work follows SURVEY.md 8(d): ops/sample = 2 * sum N_out * N_in_eff
* (G+P) (cost.hpp:71, the dense contraction count), bytes/sample = fp32 input +
output + weights once per batch.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np


@dataclass
class Workload:
    key: str
    title: str
    dims: List[int]
    G: int
    P: int
    batch: int
    std: float
    mode: str = "bspline-lut"
    lut_k: int = 8
    lut_h: int = 8
    bits_w: int = 8
    silu: bool = True
    int8_out: bool = False
    seed: int = 0
    extra: dict = field(default_factory=dict)

    def descriptor(self) -> dict:
        return {"name": self.key, "grid": {"intervals": self.G, "degree": self.P},
                "input": [self.dims[0]],
                "layers": [{"type": "linear", "n_in": a, "n_out": b}
                           for a, b in zip(self.dims, self.dims[1:])]}

    def weights(self):
        rng = np.random.default_rng(self.seed)
        nb = self.G + self.P
        Ws, Bs = [], []
        for a, b in zip(self.dims, self.dims[1:]):
            Ws.append(rng.normal(0.0, self.std, (a * nb, b)))
            Bs.append(rng.normal(0.0, 1.0 / np.sqrt(a), (a, b)) if self.silu else None)
        return Ws, Bs

    def inputs(self, rows: int, seed: int = 1) -> np.ndarray:
        rng = np.random.default_rng(self.seed * 1000 + seed)
        return rng.uniform(-1.0, 1.0, (rows, self.dims[0])).astype(np.float32)

    # -- algorithmic work --------------------------------------------
    def ops_per_sample(self) -> int:
        nb = self.G + self.P
        return int(sum(2 * b * a * nb for a, b in zip(self.dims, self.dims[1:])))

    def weight_bytes(self, layer: int) -> int:
        a, b = self.dims[layer], self.dims[layer + 1]
        nb = self.G + self.P
        esz = 2 if self.mode == "bf16" else (4 if self.mode == "fp32" else 1)
        return a * nb * b * esz + (a * b * esz if self.silu else 0)

    def layer_bytes_per_launch(self, layer: int, batch: int) -> int:
        """Algorithmic HBM bytes of one layer launch: activations in, outputs out,
        weights once.  Inputs are fp32 for layer 0; hidden activations are u16
        lattice levels on the LUT path and fp32 on the float paths."""
        lut = self.mode == "bspline-lut"
        a, b = self.dims[layer], self.dims[layer + 1]
        in_b = 4 if layer == 0 else (2 if lut else 4)
        last = layer == len(self.dims) - 2
        out_b = (1 if self.int8_out else 4) if last else (2 if lut else 4)
        return batch * (a * in_b + b * out_b) + self.weight_bytes(layer)

    def layer_ops_per_launch(self, layer: int, batch: int) -> int:
        a, b = self.dims[layer], self.dims[layer + 1]
        return 2 * batch * a * (self.G + self.P) * b


WORKLOADS = {
    # BASELINE.json configs[0]
    "c1": Workload("c1", "KAN MLP [784,64,10] G=5 P=3 batch 1024, LUT k8/h8 + int8 per-channel W",
                   [784, 64, 10], 5, 3, 1024, 0.1),
    # configs[1] -- the bench headline
    "c2": Workload("c2", "KAN MLP [784,64,10] G=5 P=3 batch 4096, LUT k8/h8 + int8 per-channel W, "
                         "SiLU base, hidden outputs requantized to the lattice, int8 logits",
                   [784, 64, 10], 5, 3, 4096, 0.1, int8_out=True),
    # configs[2]
    "c3": Workload("c3", "Wide KAN MLP [3072,1024,1024,10] G=10 P=3 batch 65536, LUT k8/h8 + int8 W",
                   [3072, 1024, 1024, 10], 10, 3, 65536, 0.05),
    "c3bf16": Workload("c3bf16", "Wide KAN MLP [3072,1024,1024,10] G=10 batch 65536, bf16 path",
                       [3072, 1024, 1024, 10], 10, 3, 65536, 0.05, mode="bf16"),
}


def get(key: str) -> Workload:
    if key not in WORKLOADS:
        raise KeyError(f"unknown workload '{key}' (have {sorted(WORKLOADS)})")
    return WORKLOADS[key]

"""The five BASELINE.json workloads, as descriptors + seeded synthetic data.

Descriptors use the reference's JSON schema (io.hpp:357-386), extended
additively for ResKAN18 (named tensors ``id`` / ``input_from`` / ``residual``
and a ``global_avgpool`` layer).  Data is synthetic with the
shapes and distributions BASELINE.json states (MNIST / CIFAR are not
available and are not used):
  inputs  ~ U[-1, 1] fp32
  spline coefficients ~ N(0, std) (0.1 for C1/C2, 0.05 for C3-C5)
  base (SiLU) weights  ~ N(0, 1/sqrt(n_in))
Algorithmic work follows SURVEY.md 8(d): ops/sample = 2 * sum N_out * N_in_eff
* (G+P) (cost.hpp:71, the dense contraction count; conv N_in_eff = K^2 C_in
per output pixel), bytes/sample = fp32 input + output + weights once per batch.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np


def walk_shapes(desc: dict) -> List[dict]:
    """Per-layer input/output shapes of a descriptor (Model::validate's walk,
    layers.hpp:252-307, with the engine's named-tensor extension)."""
    shp = list(desc["input"])
    named = {"input": shp}
    out = []
    for i, l in enumerate(desc["layers"]):
        s = named[l["input_from"]] if "input_from" in l else shp
        t = l["type"]
        if t == "linear":
            o = [l["n_out"]]
        elif t == "conv":
            k, st, p = l["kernel"], l.get("stride", 1), l.get("padding", 0)
            o = [l["c_out"], (s[1] + 2 * p - k) // st + 1, (s[2] + 2 * p - k) // st + 1]
        elif t == "maxpool":
            w = l.get("window", 2)
            o = [s[0], s[1] // w, s[2] // w]
        elif t == "global_avgpool":
            o = [s[0]]
        elif t == "flatten":
            o = [int(np.prod(s))]
        else:
            raise ValueError(t)
        out.append({"type": t, "in": s, "out": o, "layer": l})
        shp = o
        if "id" in l:
            named[l["id"]] = o
    return out


def reskan18_layers(width=(64, 128, 256, 512), n_classes=10, in_ch=3) -> list:
    """ResNet-18 topology with every conv a KAN conv: 3x3 stem, 4 stages of 2
    basic blocks, 1x1 stride-2 projection shortcuts, global average pool,
    linear classifier.  Same 20 conv + 1 linear layers, in the same order, as the
    reference's descriptors/reskan18.json, with the residual structure and the
    pooling stated explicitly."""
    L = []

    def conv(ci, co, k=3, s=1, p=1, **kw):
        d = {"type": "conv", "c_in": ci, "c_out": co, "kernel": k, "stride": s, "padding": p}
        d.update(kw)
        L.append(d)

    conv(in_ch, width[0], id="b0")
    prev, c = "b0", width[0]
    bi = 1
    for si, w in enumerate(width):
        for blk in range(2):
            down = si > 0 and blk == 0
            if down:
                conv(c, w, k=1, s=2, p=0, input_from=prev, id=f"sc{bi}")
                conv(c, w, s=2, input_from=prev)
                conv(w, w, residual=f"sc{bi}", id=f"b{bi}")
            else:
                conv(c, w, input_from=prev)
                conv(w, w, residual=prev, id=f"b{bi}")
            prev, c = f"b{bi}", w
            bi += 1
    L.append({"type": "global_avgpool"})
    L.append({"type": "linear", "n_in": width[-1], "n_out": n_classes})
    return L


@dataclass
class Workload:
    key: str
    title: str
    dims: List[int]  # MLP widths, or [input size] for descriptor-defined models
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
    # LUT-path weight scheme: 1 = per-output-channel symmetric (engine
    # extension), 0 = the reference's per-tensor asymmetric u8 (eval.hpp:70-76)
    wscheme: int = 1
    input_shape: Optional[List[int]] = None
    layers: Optional[list] = None
    extra: dict = field(default_factory=dict)

    def descriptor(self) -> dict:
        if self.layers is not None:
            d = {"name": self.key, "grid": {"intervals": self.G, "degree": self.P},
                 "input": list(self.input_shape), "layers": self.layers}
            d.update(self.extra.get("descriptor", {}))
            return d
        return {"name": self.key, "grid": {"intervals": self.G, "degree": self.P},
                "input": [self.dims[0]],
                "layers": [{"type": "linear", "n_in": a, "n_out": b}
                           for a, b in zip(self.dims, self.dims[1:])]}

    def eval_options(self) -> dict:
        """EvalOptions keyword arguments of this workload (engine.EvalOptions);
        int8 logits additionally need the output scale the bench calibrates."""
        return dict(mode=self.mode, lut_k=self.lut_k, lut_h=self.lut_h, bits_w=self.bits_w,
                    w_scheme=self.wscheme, silu_base=self.silu)

    def scheme(self) -> str:
        """One-line statement of the arithmetic this workload runs."""
        if self.mode != "bspline-lut":
            return f"{self.mode} path" + (", SiLU base term" if self.silu else "")
        w = ("per-tensor asymmetric u8 W (the reference scheme, eval.hpp:70-76)" if self.wscheme == 0
             else f"per-channel symmetric int{self.bits_w} W")
        return (f"LUT k{self.lut_k}/h{self.lut_h}, {w}, " + ("SiLU base term" if self.silu else "no SiLU term")
                + (", int8 logits" if self.int8_out else ", fp32 logits"))

    @property
    def reference_scheme(self) -> bool:
        """True when the reference's own CPU path computes this exact arithmetic
        (bspline-lut, per-tensor u8 W, no SiLU, fp32 logits)."""
        return (self.mode == "bspline-lut" and self.wscheme == 0 and not self.silu and not self.int8_out
                and self.bits_w == 8)

    def kan_layers(self) -> List[dict]:
        """KAN layers in order: reference inputs (conv: K^2 C_in), outputs, output
        pixels per sample, and input / output elements per sample."""
        res = []
        for s in walk_shapes(self.descriptor()):
            l = s["layer"]
            if s["type"] == "linear":
                res.append({"n_in": l["n_in"], "n_out": l["n_out"], "pix": 1,
                            "in_elems": int(np.prod(s["in"])), "out_elems": l["n_out"]})
            elif s["type"] == "conv":
                pix = s["out"][1] * s["out"][2]
                res.append({"n_in": l["kernel"] ** 2 * l["c_in"], "n_out": l["c_out"], "pix": pix,
                            "in_elems": int(np.prod(s["in"])), "out_elems": int(np.prod(s["out"]))})
        return res

    @property
    def n_kan(self) -> int:
        return len(self.kan_layers())

    @property
    def out_size(self) -> int:
        """Values per sample of the model output (the last layer, flattened)."""
        return int(np.prod(walk_shapes(self.descriptor())[-1]["out"]))

    @property
    def reference_expressible(self) -> bool:
        """True when the reference's own model_forward can run this model: no
        engine descriptor extensions, and a flat (linear) output layer
        (model_forward returns flat logits, eval.hpp:200-253)."""
        d = self.descriptor()
        ext = {"id", "input_from", "residual"}
        return d["layers"][-1]["type"] == "linear" and "conv_output" not in d and all(
            l["type"] != "global_avgpool" and not (ext & set(l)) for l in d["layers"])

    @property
    def input_size(self) -> int:
        return int(np.prod(self.input_shape)) if self.input_shape else self.dims[0]

    def weights(self):
        rng = np.random.default_rng(self.seed)
        nb = self.G + self.P
        Ws, Bs = [], []
        for kl in self.kan_layers():
            a, b = kl["n_in"], kl["n_out"]
            Ws.append(rng.normal(0.0, self.std, (a * nb, b)))
            Bs.append(rng.normal(0.0, 1.0 / np.sqrt(a), (a, b)) if self.silu else None)
        return Ws, Bs

    def inputs(self, rows: int, seed: int = 1) -> np.ndarray:
        rng = np.random.default_rng(self.seed * 1000 + seed)
        return rng.uniform(-1.0, 1.0, (rows, self.input_size)).astype(np.float32)

    # -- algorithmic work --------------------------------------------
    def ops_per_sample(self) -> int:
        nb = self.G + self.P
        return int(sum(2 * kl["pix"] * kl["n_in"] * nb * kl["n_out"] for kl in self.kan_layers()))

    def weight_bytes(self, layer: int) -> int:
        kl = self.kan_layers()[layer]
        a, b = kl["n_in"], kl["n_out"]
        if self.mode == "spline-table":  # u8 tables [n_in][2^bits_a][n_out]
            return a * b << self.lut_k
        nb = self.G + self.P
        esz = 2 if self.mode == "bf16" else (4 if self.mode == "fp32" else 1)
        return a * nb * b * esz + (a * b * esz if self.silu else 0)

    def layer_bytes_per_launch(self, layer: int, batch: int) -> int:
        """Algorithmic HBM bytes of one layer launch: activations in, outputs out,
        weights once.  Inputs are fp32 for layer 0; hidden activations are u16
        lattice levels on the LUT path and fp32 on the float paths."""
        lut = self.mode == "bspline-lut"
        st = self.mode == "spline-table"  # hidden tensors are u8 input levels
        kls = self.kan_layers()
        kl = kls[layer]
        in_b = 4 if layer == 0 else (1 if st else (2 if lut else 4))
        last = layer == len(kls) - 1
        out_b = (1 if self.int8_out else 4) if last else (1 if st else (2 if lut else 4))
        return batch * (kl["in_elems"] * in_b + kl["out_elems"] * out_b) + self.weight_bytes(layer)

    def layer_ops_per_launch(self, layer: int, batch: int) -> int:
        kl = self.kan_layers()[layer]
        if self.mode == "spline-table":  # one table lookup + one integer add per connection
            return batch * kl["pix"] * kl["n_in"] * kl["n_out"]
        return 2 * batch * kl["pix"] * kl["n_in"] * (self.G + self.P) * kl["n_out"]


WORKLOADS = {
    # BASELINE.json configs[0]
    "c1": Workload("c1", "KAN MLP [784,64,10] G=5 P=3 batch 1024, LUT k8/h8 + int8 per-channel W",
                   [784, 64, 10], 5, 3, 1024, 0.1),
    # configs[1] -- the bench headline
    "c2": Workload("c2", "KAN MLP [784,64,10] G=5 P=3 batch 4096, LUT k8/h8 + int8 per-channel W, "
                         "SiLU base, hidden outputs requantized to the lattice, int8 logits",
                   [784, 64, 10], 5, 3, 4096, 0.1, int8_out=True),
    # configs[0], the float accuracy baseline on the same model: fp32 Cox-de Boor
    # basis + fp32 FFMA contraction (the paper's LUT-vs-recursion comparison,
    # PAPER.md:603)
    "c1fp32": Workload("c1fp32", "KAN MLP [784,64,10] G=5 P=3 batch 1024, fp32 Cox-de Boor path",
                       [784, 64, 10], 5, 3, 1024, 0.1, mode="fp32"),
    # configs[1] sweep points (sweep.hpp:112-119 enumerates the k/h cross
    # product; "no GPU benefit below 8 bits")
    "c2k4": Workload("c2k4", "KAN MLP [784,64,10] G=5 P=3 batch 4096, LUT k4/h4 + int8 per-channel W, "
                             "SiLU base, int8 logits", [784, 64, 10], 5, 3, 4096, 0.1, lut_k=4, lut_h=4,
                     int8_out=True),
    "c2k3": Workload("c2k3", "KAN MLP [784,64,10] G=5 P=3 batch 4096, LUT k3/h3 + int8 per-channel W, "
                             "SiLU base, int8 logits", [784, 64, 10], 5, 3, 4096, 0.1, lut_k=3, lut_h=3,
                     int8_out=True),
    "c2k2": Workload("c2k2", "KAN MLP [784,64,10] G=5 P=3 batch 4096, LUT k2/h2 + int8 per-channel W, "
                             "SiLU base, int8 logits", [784, 64, 10], 5, 3, 4096, 0.1, lut_k=2, lut_h=2,
                     int8_out=True),
    "c2w4": Workload("c2w4", "KAN MLP [784,64,10] G=5 P=3 batch 4096, LUT k8/h8 + int4 per-channel W, "
                             "SiLU base, int8 logits", [784, 64, 10], 5, 3, 4096, 0.1, bits_w=4, int8_out=True),
    # configs[2]
    "c3": Workload("c3", "Wide KAN MLP [3072,1024,1024,10] G=10 P=3 batch 65536, LUT k8/h8 + int8 W",
                   [3072, 1024, 1024, 10], 10, 3, 65536, 0.05),
    "c3bf16": Workload("c3bf16", "Wide KAN MLP [3072,1024,1024,10] G=10 batch 65536, bf16 path",
                       [3072, 1024, 1024, 10], 10, 3, 65536, 0.05, mode="bf16"),
    # configs[3]
    "c4": Workload("c4", "KAN conv 3x3 s1 p1 64->64 on 32x32, G=5 P=3 batch 256, LUT k8/h8 + int8 W "
                         "(implicit im2col)",
                   [64 * 32 * 32], 5, 3, 256, 0.05, input_shape=[64, 32, 32],
                   layers=[{"type": "conv", "c_in": 64, "c_out": 64, "kernel": 3, "stride": 1,
                            "padding": 1}]),
    # configs[4] -- the bench headline (BASELINE metric "at 1/2/4/8 B200" is
    # quoted on this config).  "3-bit B-spline table + int8 coeffs": run in the
    # reference's own weight scheme (per-tensor asymmetric 8-bit codes, no SiLU
    # term, fp32 logits), so the reference's CPU path computes the same numbers
    "c5": Workload("c5", "ResKAN18 (ResNet-18 topology, KAN convs) on 3x32x32, G=5 P=3 batch 8192, "
                         "LUT k8/h3 (3-bit table) + 8-bit W",
                   [3 * 32 * 32], 5, 3, 8192, 0.05, lut_h=3, input_shape=[3, 32, 32], silu=False,
                   wscheme=0, layers=reskan18_layers(), extra={"descriptor": {"conv_output": "floor"}}),
    # the same network with per-channel int8 W and the SiLU base term (engine extensions)
    "c5pc": Workload("c5pc", "ResKAN18 on 3x32x32, G=5 P=3 batch 8192, LUT k8/h3 + per-channel int8 W, "
                             "SiLU base term",
                     [3 * 32 * 32], 5, 3, 8192, 0.05, lut_h=3, input_shape=[3, 32, 32],
                     layers=reskan18_layers(), extra={"descriptor": {"conv_output": "floor"}}),
    # spline-table mode (spline_table.hpp) on the C1/C2/C4
    # shapes, 256-entry 8-bit tables (bits_a = 8, h = 8), no SiLU term (the
    # reference's tables replace the whole activation phi_{i,j})
    "c1st": Workload("c1st", "KAN MLP [784,64,10] G=5 P=3 batch 1024, spline tables bits_a=8 h=8",
                     [784, 64, 10], 5, 3, 1024, 0.1, mode="spline-table", silu=False),
    "c2st": Workload("c2st", "KAN MLP [784,64,10] G=5 P=3 batch 4096, spline tables bits_a=8 h=8",
                     [784, 64, 10], 5, 3, 4096, 0.1, mode="spline-table", silu=False),
    "c2st4": Workload("c2st4", "KAN MLP [784,64,10] G=5 P=3 batch 4096, spline tables bits_a=4 h=4",
                      [784, 64, 10], 5, 3, 4096, 0.1, mode="spline-table", lut_k=4, lut_h=4,
                      silu=False),
    "c4st": Workload("c4st", "KAN conv 3x3 s1 p1 64->64 on 32x32, G=5 P=3 batch 256, spline tables "
                             "bits_a=8 h=8 (implicit im2col)",
                     [64 * 32 * 32], 5, 3, 256, 0.05, mode="spline-table", silu=False,
                     input_shape=[64, 32, 32],
                     layers=[{"type": "conv", "c_in": 64, "c_out": 64, "kernel": 3, "stride": 1,
                              "padding": 1}]),
}


def get(key: str) -> Workload:
    if key not in WORKLOADS:
        raise KeyError(f"unknown workload '{key}' (have {sorted(WORKLOADS)})")
    return WORKLOADS[key]

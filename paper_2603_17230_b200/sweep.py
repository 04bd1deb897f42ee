"""GPU backend for the reference's accuracy sweep (sweep.hpp:97-408).

Mirrors the reference's names and semantics:

  enumerate_configs(spec)     sweep.hpp:97-130  (stable Cartesian order; table modes
                                                 drop unrealizable bit widths)
  evaluate_accuracy(...)      eval.hpp:279-287  (kan_engine_evaluate_accuracy)
  run_sweep(...)              sweep.hpp:230-316 (accuracy + analytic costs per config)
  pareto_front(score, cost)   sweep.hpp:145-165
  csv_header / csv_row        sweep.hpp:190-210

Every configuration is evaluated on the GPU by reconfiguring one engine:
fake-quant -> KAN_MODE_FAKE_QUANT, bspline-lut -> KAN_MODE_BSPLINE_LUT with the
reference's per-tensor weights, spline-table -> KAN_MODE_SPLINE_TABLE.  A
configuration the engine cannot realize (e.g. passthrough activations with a
quantized basis, or fp64 weights on the integer LUT path) is reported with
accuracy NaN and its reason, never silently evaluated elsewhere.
The caller passes the evaluation rows (the reference draws a seeded subset
first, sweep.hpp:236-237).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import configs as _configs
from .engine import Engine, EvalOptions, W_PER_TENSOR_ASYM

PASSTHROUGH = 32


@dataclass
class SweepSpec:
    bits_w_set: List[int] = field(default_factory=lambda: [PASSTHROUGH])
    bits_a_set: List[int] = field(default_factory=lambda: [PASSTHROUGH])
    bits_b_set: List[int] = field(default_factory=lambda: [PASSTHROUGH])
    modes: List[str] = field(default_factory=lambda: ["fake-quant"])


@dataclass
class SweepConfig:
    mode: str
    bits_w: int = PASSTHROUGH
    bits_a: int = PASSTHROUGH
    bits_b: int = PASSTHROUGH


@dataclass
class ParetoPoint:
    config: SweepConfig
    accuracy: float = 0.0
    bitops: int = 0
    lut_mem_bits: int = 0
    spline_mem_bits: int = 0
    fp32_coeff_bits: int = 0
    note: str = ""


def enumerate_configs(spec: SweepSpec) -> List[SweepConfig]:
    """sweep.hpp:97-130."""
    if not (spec.bits_w_set and spec.bits_a_set and spec.bits_b_set and spec.modes):
        raise ValueError("enumerate_configs: empty bit-width or mode set")
    out = []
    for mode in spec.modes:
        if mode == "fake-quant":
            out += [SweepConfig(mode, w, a, b) for w in spec.bits_w_set for a in spec.bits_a_set
                    for b in spec.bits_b_set]
        elif mode == "bspline-lut":
            out += [SweepConfig(mode, w, a, b) for w in spec.bits_w_set for a in spec.bits_a_set
                    if 1 <= a <= 8 for b in spec.bits_b_set if 2 <= b <= 8]
        elif mode == "spline-table":
            out += [SweepConfig(mode, PASSTHROUGH, a, b) for a in spec.bits_a_set if 1 <= a <= 8
                    for b in spec.bits_b_set if 2 <= b <= 8]
        else:
            raise ValueError(f"enumerate_configs: unknown mode '{mode}'")
    return out


# ---- analytic costs (cost.hpp:15-130) ------------------------------------------
def arch_layers(desc: dict):
    """ArchLayer list of a descriptor (arch_of, cost.hpp:168-211)."""
    out = []
    for s in _configs.walk_shapes(desc):
        l = s["layer"]
        if s["type"] == "linear":
            out.append({"eff_n_in": l["n_in"], "eff_n_out": l["n_out"], "connections": l["n_in"] * l["n_out"]})
        elif s["type"] == "conv":
            k, ho, wo = l["kernel"], s["out"][1], s["out"][2]
            out.append({"eff_n_in": k * k * l["c_in"] * ho * wo, "eff_n_out": l["c_out"],
                        "connections": k * k * l["c_in"] * l["c_out"]})
    return out


def recursion_mul_factor(G: int, P: int) -> int:
    return 4 * (P * (G + 2 * P) - P * (P - 1) // 2)


def bitops_kan(desc, bits_w, bits_a, bits_b, batch=1, tabulated=False) -> int:
    G, P = desc["grid"]["intervals"], desc["grid"]["degree"]
    tot = 0
    for l in arch_layers(desc):
        matmul = batch * l["eff_n_out"] * l["eff_n_in"] * (G + P)
        bspline = batch * l["eff_n_in"] * recursion_mul_factor(G, P)
        tot += matmul * bits_b * bits_w + (0 if tabulated else bspline * bits_a * bits_a)
    return tot


def lut_memory_bits(P: int, k: int, h: int) -> int:
    return (1 << k) * ((P + 2) // 2) * h


def spline_table_bits(desc, bits_a: int, h: int) -> int:
    return sum(l["connections"] for l in arch_layers(desc)) * (1 << bits_a) * h


def fp32_coeff_bits(desc) -> int:
    G, P = desc["grid"]["intervals"], desc["grid"]["degree"]
    return sum(l["connections"] for l in arch_layers(desc)) * (G + P) * 32


def fill_costs(p: ParetoPoint, desc: dict):
    """detail::fill_costs, sweep.hpp:171-188."""
    c = p.config
    p.fp32_coeff_bits = fp32_coeff_bits(desc)
    if c.mode == "fake-quant":
        p.bitops = bitops_kan(desc, c.bits_w, c.bits_a, c.bits_b, 1, False)
    elif c.mode == "bspline-lut":
        p.bitops = bitops_kan(desc, c.bits_w, c.bits_a, c.bits_b, 1, True)
        p.lut_mem_bits = lut_memory_bits(desc["grid"]["degree"], c.bits_a, c.bits_b)
    else:
        p.spline_mem_bits = spline_table_bits(desc, c.bits_a, c.bits_b)


def pareto_front(score: Sequence[float], cost: Sequence[float]) -> List[int]:
    """sweep.hpp:145-165: indices of the non-dominated points (max score, min cost)."""
    if len(score) != len(cost):
        raise ValueError("pareto_front: length mismatch")
    if not score:
        raise ValueError("pareto_front: empty input")
    keep = []
    for p in range(len(score)):
        dominated = any(q != p and score[q] >= score[p] and cost[q] <= cost[p]
                        and (score[q] > score[p] or cost[q] < cost[p]) for q in range(len(score)))
        if not dominated:
            keep.append(p)
    return keep


def csv_header() -> str:
    return ("model,mode,bw_w,bw_a,bw_b,accuracy,bitops,lut_mem_bits,spline_mem_bits,"
            "fp32_coeff_bits")


def csv_row(model_name: str, p: ParetoPoint) -> str:
    c = p.config
    return (f"{model_name},{c.mode},{c.bits_w},{c.bits_a},{c.bits_b},{p.accuracy:.17g},{p.bitops},"
            f"{p.lut_mem_bits},{p.spline_mem_bits},{p.fp32_coeff_bits}")


def eval_options(c: SweepConfig) -> EvalOptions:
    """The engine configuration of one sweep point (sweep.hpp:258-276)."""
    if c.mode == "fake-quant":
        return EvalOptions(mode="fake-quant", bits_w=c.bits_w, lut_k=c.bits_a, lut_h=c.bits_b)
    if c.mode == "bspline-lut":
        return EvalOptions(mode="bspline-lut", lut_k=c.bits_a, lut_h=c.bits_b, bits_w=c.bits_w,
                           w_scheme=W_PER_TENSOR_ASYM)
    return EvalOptions(mode="spline-table", lut_k=c.bits_a, lut_h=c.bits_b)


def run_sweep(engine: Engine, x, labels, spec: SweepSpec, desc: Optional[dict] = None):
    """run_sweep (sweep.hpp:230-316) on the GPU: every configuration's top-1
    accuracy on (x, labels) -- CUDA tensors, fp32 [n, input_size] and int32 [n] --
    plus its analytic costs; returns (points, pareto_bitops, pareto_memory)."""
    desc = desc or engine.descriptor
    points = []
    for c in enumerate_configs(spec):
        p = ParetoPoint(c)
        try:
            engine.configure(eval_options(c))
            p.accuracy = engine.evaluate_accuracy(x, labels)
        except NotImplementedError as ex:
            p.accuracy, p.note = math.nan, f"unsupported on the GPU: {ex}"
        except ValueError as ex:
            p.accuracy, p.note = math.nan, f"invalid: {ex}"
        fill_costs(p, desc)
        points.append(p)
    ok = [i for i, p in enumerate(points) if not math.isnan(p.accuracy)]
    pb = [ok[i] for i in pareto_front([points[i].accuracy for i in ok],
                                      [points[i].bitops for i in ok])] if ok else []
    wt = [i for i in ok if points[i].lut_mem_bits + points[i].spline_mem_bits > 0]
    pm = [wt[i] for i in pareto_front([points[i].accuracy for i in wt],
                                      [points[i].lut_mem_bits + points[i].spline_mem_bits
                                       for i in wt])] if wt else []
    return points, pb, pm

"""B200-native KAN inference engine (KANtize hot path: the KAN layer forward).

The compute lives in ``libkan_b200.so`` (CUDA for sm_100a behind the C ABI in
``include/kan_b200.h``); :mod:`paper_2603_17230_b200.engine` mirrors the
reference's evaluation interface over it.

The engine names are resolved lazily: ``import paper_2603_17230_b200.configs``
(workload descriptors and seeded data, pure numpy) does not load the shared
library, so the bench's reference arm runs without mapping any of this repo's
native code.  Touching any engine name loads ``libkan_b200.so`` and raises if
it is missing (there is no CPU fallback).
"""
from __future__ import annotations

import importlib

_ENGINE_NAMES = frozenset((
    "Engine", "EvalOptions", "KanError", "build_bspline_lut", "eval_mode_from_string",
    "kan_linear_forward", "tabulated_kan_forward", "lattice_thresholds", "MODE_FP32", "MODE_BF16",
    "MODE_BSPLINE_LUT", "MODE_SPLINE_TABLE", "build_spline_tables", "spline_table_forward",
    "spline_thresholds", "load_container", "save_container", "crc32", "W_PER_TENSOR_ASYM",
    "W_PER_CHANNEL_SYM", "OUT_F32", "OUT_I8", "PASSTHROUGH_BITS", "LIB_PATH", "forward_sharded",
))

__all__ = sorted(_ENGINE_NAMES)


def __getattr__(name):
    if name in _ENGINE_NAMES:
        return getattr(importlib.import_module(".engine", __name__), name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")

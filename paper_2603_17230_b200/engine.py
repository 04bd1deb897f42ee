"""Python mirror of the reference's KAN evaluation interface over the C ABI.

The reference (proj/include/kantize/) exposes

  model_from_descriptor(json) -> Model                io.hpp:357-386
  model_forward(model, inputs, EvalOptions)            eval.hpp:200-253
  predict(model, inputs, EvalOptions, chunk=256)       eval.hpp:255-276
  tabulated_kan_forward(acts, layer, lut, bits_w)      lut.hpp:217-231
  kan_linear_forward(acts, layer)                      layers.hpp:118-121
  build_bspline_lut(P, k, h)                           lut.hpp:103-131
  build_spline_tables(layer, bits_a, h)                spline_table.hpp:87-95
  spline_table_forward(acts, tables)                   spline_table.hpp:90-107
  eval_mode_from_string("fp32" | "bspline-lut" ...)    eval.hpp:19-25

This module keeps those names and argument meanings, but every forward runs in
``libkan_b200.so`` (include/kan_b200.h) on a CUDA device.  There is no CPU
fallback: if the shared library is missing, importing this module raises.
torch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkan_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        " (the engine has no CPU fallback)")

_lib = C.CDLL(LIB_PATH)

KAN_OK = 0
_STATUS = {
    1: ValueError, 2: ValueError, 3: IndexError, 4: RuntimeError, 5: RuntimeError,
    6: OSError, 7: ValueError, 8: ValueError, 9: NotImplementedError, 10: RuntimeError,
}
STATUS_NAMES = {0: "OK", 1: "INVALID_ARGUMENT", 2: "SHAPE_MISMATCH", 3: "OUT_OF_RANGE",
                4: "CUDA", 5: "NCCL", 6: "IO", 7: "FORMAT", 8: "CHECKSUM", 9: "UNSUPPORTED",
                10: "LOGIC"}

MODE_FP32, MODE_BF16, MODE_BSPLINE_LUT, MODE_SPLINE_TABLE, MODE_FAKE_QUANT = 0, 1, 2, 3, 4
W_PER_TENSOR_ASYM, W_PER_CHANNEL_SYM = 0, 1
OUT_F32, OUT_I8 = 0, 1
PASSTHROUGH_BITS = 32  # quant.hpp:15


class KanError(Exception):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{STATUS_NAMES.get(status, status)}] {msg}")
        self.status = status


class _Config(C.Structure):
    _fields_ = [("mode", C.c_int), ("lut_k", C.c_int), ("lut_h", C.c_int), ("bits_w", C.c_int),
                ("w_scheme", C.c_int), ("silu_base", C.c_int), ("out_kind", C.c_int),
                ("out_scale", C.c_double), ("split_k", C.c_int)]


_vp = C.c_void_p
_lib.kan_engine_create.argtypes = [C.c_char_p, C.c_int, C.POINTER(_vp)]
_lib.kan_engine_destroy.argtypes = [_vp]
_lib.kan_engine_last_error.argtypes = [_vp]
_lib.kan_engine_last_error.restype = C.c_char_p
_lib.kan_engine_num_kan_layers.argtypes = [_vp]
_lib.kan_engine_input_size.argtypes = [_vp]
_lib.kan_engine_input_size.restype = C.c_int64
_lib.kan_engine_output_count.argtypes = [_vp]
_lib.kan_engine_layer_shape.argtypes = [_vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
_lib.kan_engine_set_coeffs.argtypes = [_vp, C.c_int, _vp, C.c_int64, _vp, C.c_int64]
_lib.kan_engine_configure.argtypes = [_vp, C.POINTER(_Config)]
_lib.kan_engine_forward.argtypes = [_vp, _vp, C.c_int64, _vp, _vp]
_lib.kan_engine_forward_host.argtypes = [_vp, _vp, C.c_int64, _vp, _vp]
_lib.kan_engine_predict.argtypes = [_vp, _vp, C.c_int64, _vp, _vp]
_lib.kan_engine_evaluate_accuracy.argtypes = [_vp, _vp, _vp, C.c_int64, C.POINTER(C.c_double), _vp]
_lib.kan_engine_layer_levels.argtypes = [_vp, C.c_int, _vp, C.c_int64, _vp, _vp]
_lib.kan_engine_layer_accumulators.argtypes = [_vp, C.c_int, _vp, C.c_int64, _vp, _vp, _vp]
_lib.kan_engine_lut.argtypes = [_vp, _vp, C.c_int64]
_lib.kan_engine_lut.restype = C.c_int64
_lib.kan_engine_last_launches.argtypes = [_vp]
_lib.kan_engine_set_profiling.argtypes = [_vp, C.c_int]
_lib.kan_engine_layer_time_ms.argtypes = [_vp, C.c_int, C.POINTER(C.c_double),
                                          C.POINTER(C.c_int64)]
_lib.kan_engine_layer_timeline.argtypes = [_vp, C.c_int, _vp, C.c_int64]
_lib.kan_engine_layer_timeline.restype = C.c_int64
_lib.kan_engine_set_activation_ranges.argtypes = [_vp, _vp, C.c_int]
_lib.kan_engine_linear_backward.argtypes = [_vp, C.c_int, _vp, C.c_int64, _vp, _vp, _vp, _vp]
_lib.kan_engine_sgd_step.argtypes = [_vp, C.c_int, _vp, C.c_double, C.c_double, _vp]
_lib.kan_engine_get_coeffs.argtypes = [_vp, C.c_int, _vp, C.c_int64]
_lib.kan_softmax_cross_entropy.argtypes = [_vp, _vp, C.c_int64, C.c_int, _vp, _vp, _vp]
_lib.kan_engine_conv_backward.argtypes = [_vp, C.c_int, _vp, C.c_int64, _vp, _vp, _vp, _vp]
_lib.kan_maxpool2_f32.argtypes = [_vp, C.c_int64, C.c_int, C.c_int, C.c_int, _vp, _vp]
_lib.kan_maxpool2_backward_f32.argtypes = [_vp, C.c_int64, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp]
_lib.kan_engine_set_spline_tables.argtypes = [_vp, C.c_int, _vp, C.c_int64, C.c_int, C.c_int, _vp, _vp]
_lib.kan_engine_spline_table.argtypes = [_vp, C.c_int, _vp, C.c_int64, _vp, _vp]
_lib.kan_engine_spline_table.restype = C.c_int64
_lib.kan_container_load.argtypes = [C.c_char_p, C.POINTER(_vp)]
_lib.kan_container_destroy.argtypes = [_vp]
_lib.kan_container_last_error.argtypes = [_vp]
_lib.kan_container_last_error.restype = C.c_char_p
_lib.kan_container_descriptor.argtypes = [_vp]
_lib.kan_container_descriptor.restype = C.c_char_p
_lib.kan_container_num_kan_layers.argtypes = [_vp]
_lib.kan_container_coeffs.argtypes = [_vp, C.c_int, _vp, C.c_int64]
_lib.kan_container_coeffs.restype = C.c_int64
_lib.kan_container_lut.argtypes = [_vp, _vp, C.c_int64, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                   C.POINTER(C.c_int)]
_lib.kan_container_lut.restype = C.c_int64
_lib.kan_container_num_spline_tables.argtypes = [_vp]
_lib.kan_container_spline_table.argtypes = [_vp, C.c_int, _vp, C.c_int64, C.POINTER(C.c_int),
                                            C.POINTER(C.c_int), _vp, _vp]
_lib.kan_container_spline_table.restype = C.c_int64
_lib.kan_container_save.argtypes = [C.c_char_p, C.c_char_p, _vp, _vp, C.c_int64, C.c_int, C.c_int,
                                    _vp, C.c_int, C.c_int, _vp, _vp]
_lib.kan_container_save_error.restype = C.c_char_p
_lib.kan_crc32.argtypes = [_vp, C.c_size_t]
_lib.kan_crc32.restype = C.c_uint32
_lib.kan_engine_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(_vp)]
_lib.kan_lut_build.argtypes = [C.c_int, C.c_int, C.c_int, _vp, C.c_int64]
_lib.kan_lut_build.restype = C.c_int64
_lib.kan_lattice_thresholds.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _vp,
                                        C.c_int64]
_lib.kan_lattice_thresholds.restype = C.c_int64
_lib.kan_spline_thresholds.argtypes = [C.c_double, C.c_double, C.c_int, _vp, C.c_int64]
_lib.kan_spline_thresholds.restype = C.c_int64
_lib.kan_engine_set_option.argtypes = [_vp, C.c_int, C.c_int64]
_lib.kan_engine_last_plan.argtypes = [_vp]
_lib.kan_engine_last_plan.restype = C.c_char_p
_lib.kan_engine_forward_sharded.argtypes = [_vp, C.c_int, _vp, C.c_int64, _vp, _vp]
_lib.kan_engine_forward_sharded_host.argtypes = [_vp, C.c_int, _vp, C.c_int64, _vp]
_lib.kan_shard_rows.argtypes = [C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
_lib.kan_shard_rows.restype = None

# kan_option (include/kan_b200.h): tuning / debug switches, no environment reads
OPTIONS = {"no_conv3": 1, "no_im2col": 2, "force_bn": 3, "tables": 4, "epi_stage": 5, "conv3_mc": 6,
           "lv_sidecar": 7, "level_prepass_min": 8, "st_prepass": 9, "st_slices": 10, "timeline": 11,
           "force_nacc1": 12, "record_plan": 13, "dbg_flags": 14, "no_convw": 15,
           "convw_rings": 16, "convw_tr": 17, "convw_mc": 18, "convw_bn": 19, "convw_lock": 20, "no_fuse": 21, "fuse_persistent": 22, "convw_no_kym": 23, "convw_dual": 24}

# exported symbols declared in include/kan_b200.h (checked by the CPU tests)
EXPORTED = [
    "kan_engine_create", "kan_engine_destroy", "kan_engine_last_error",
    "kan_engine_num_kan_layers", "kan_engine_input_size", "kan_engine_output_count",
    "kan_engine_layer_shape", "kan_engine_set_coeffs", "kan_engine_configure",
    "kan_engine_forward", "kan_engine_forward_host", "kan_engine_predict",
    "kan_engine_layer_levels", "kan_engine_layer_accumulators", "kan_engine_lut",
    "kan_engine_last_launches", "kan_lut_build", "kan_lattice_thresholds",
    "kan_engine_set_profiling", "kan_engine_layer_time_ms", "kan_engine_layer_timeline",
    "kan_engine_set_spline_tables", "kan_engine_spline_table", "kan_spline_thresholds",
    "kan_container_load", "kan_container_destroy", "kan_container_last_error",
    "kan_container_descriptor", "kan_container_num_kan_layers", "kan_container_coeffs",
    "kan_container_lut", "kan_container_num_spline_tables", "kan_container_spline_table",
    "kan_container_save", "kan_container_save_error", "kan_crc32", "kan_engine_load",
    "kan_engine_evaluate_accuracy", "kan_engine_set_activation_ranges",
    "kan_engine_linear_backward", "kan_softmax_cross_entropy", "kan_engine_conv_backward",
    "kan_maxpool2_f32", "kan_maxpool2_backward_f32", "kan_engine_set_option", "kan_engine_last_plan",
    "kan_engine_forward_sharded", "kan_engine_forward_sharded_host", "kan_shard_rows",
    "kan_engine_sgd_step", "kan_engine_get_coeffs",
]


def shard_rows(batch: int, g: int, n: int):
    """[start, stop) rows of shard g of n (kan_shard_rows: contiguous, ceil(batch/n) each)."""
    a, b = C.c_int64(), C.c_int64()
    _lib.kan_shard_rows(batch, g, n, C.byref(a), C.byref(b))
    return a.value, b.value


def _group_error(engines, st):
    msg = _lib.kan_engine_last_error(engines[0]._h).decode()
    raise _STATUS.get(st, RuntimeError)(KanError(st, msg))


def forward_sharded(engines, x_shards, out, streams=None):
    """kan_engine_forward_sharded: engines[g] (one per device, or several on one)
    runs rows shard_rows(batch, g, n) from x_shards[g] (a CUDA tensor on its
    device); the logits land in `out` ([batch, output_count] on engines[0]'s
    device).  Returns `out`; streams[0] (default: device 0's current stream)
    waits for every shard."""
    torch = _torch()
    n = len(engines)
    batch = out.shape[0]
    hs = (_vp * n)(*[e._h for e in engines])
    xs = (_vp * n)(*[(x.data_ptr() if x is not None and x.numel() else None) for x in x_shards])
    if streams is None:
        streams = [torch.cuda.current_stream(e.device) for e in engines]
    ss = (_vp * n)(*[s.cuda_stream for s in streams])
    st = _lib.kan_engine_forward_sharded(hs, n, xs, batch, out.data_ptr(), ss)
    if st != KAN_OK:
        _group_error(engines, st)
    return out


def forward_sharded_host(engines, x: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
    """kan_engine_forward_sharded_host: host rows in, host logits out; every
    shard's H2D copy, forward and D2H copy runs on its engine's own stream."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    e0 = engines[0]
    i8 = e0.opts is not None and e0.opts.out_kind == OUT_I8
    if out is None:
        out = np.empty((x.shape[0], e0.output_count), dtype=np.int8 if i8 else np.float32)
    n = len(engines)
    hs = (_vp * n)(*[e._h for e in engines])
    st = _lib.kan_engine_forward_sharded_host(hs, n, x.ctypes.data, x.shape[0], out.ctypes.data)
    if st != KAN_OK:
        _group_error(engines, st)
    return out


def lattice_thresholds(G: int, P: int, k: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """The engine's exact fp32 level thresholds (host utility, no GPU)."""
    n = _lib.kan_lattice_thresholds(G, P, lo, hi, k, None, 0)
    if n < 0:
        raise ValueError("lattice_thresholds: bad arguments")
    out = np.zeros(n, dtype=np.float32)
    _lib.kan_lattice_thresholds(G, P, lo, hi, k, out.ctypes.data, n)
    return out


def spline_thresholds(bits_a: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """The engine's exact fp32 spline-table input level thresholds (host utility)."""
    n = _lib.kan_spline_thresholds(lo, hi, bits_a, None, 0)
    if n < 0:
        raise ValueError("spline_thresholds: bad arguments")
    out = np.zeros(n, dtype=np.float32)
    _lib.kan_spline_thresholds(lo, hi, bits_a, out.ctypes.data, n)
    return out


def crc32(data: bytes) -> int:
    """crc32 of io.hpp:31-45."""
    buf = (C.c_uint8 * max(len(data), 1)).from_buffer_copy(data or b"\0")
    return _lib.kan_crc32(C.addressof(buf), len(data))


def load_container(path: str) -> dict:
    """load_container (io.hpp:217-350): the model as a descriptor, its coefficients,
    and the LUT / spline tables stored with it.  Raises OSError (io_error),
    ValueError (format_error / checksum_error; KanError.status tells which)."""
    h = _vp()
    st = _lib.kan_container_load(str(path).encode(), C.byref(h))
    try:
        if st != KAN_OK:
            msg = _lib.kan_container_last_error(h).decode()
            raise _STATUS.get(st, RuntimeError)(KanError(st, msg))
        out = {"descriptor": json.loads(_lib.kan_container_descriptor(h).decode()), "coeffs": [],
               "lut": None, "spline_tables": []}
        for i in range(_lib.kan_container_num_kan_layers(h)):
            n = _lib.kan_container_coeffs(h, i, None, 0)
            w = np.zeros(n)
            _lib.kan_container_coeffs(h, i, w.ctypes.data, n)
            out["coeffs"].append(w)
        deg, k, hb = C.c_int(), C.c_int(), C.c_int()
        n = _lib.kan_container_lut(h, None, 0, C.byref(deg), C.byref(k), C.byref(hb))
        if n > 0:
            e = np.zeros(n, dtype=np.uint8)
            _lib.kan_container_lut(h, e.ctypes.data, n, None, None, None)
            out["lut"] = {"entries": e, "degree": deg.value, "k": k.value, "h": hb.value}
        for t in range(_lib.kan_container_num_spline_tables(h)):
            ba, hv = C.c_int(), C.c_int()
            qd, qi = np.zeros(2), np.zeros(4, dtype=np.int64)
            n = _lib.kan_container_spline_table(h, t, None, 0, None, None, None, None)
            v = np.zeros(n, dtype=np.uint8)
            _lib.kan_container_spline_table(h, t, v.ctypes.data, n, C.byref(ba), C.byref(hv),
                                            qd.ctypes.data, qi.ctypes.data)
            out["spline_tables"].append({"values": v, "bits_a": ba.value, "h": hv.value,
                                         "qp_d": qd, "qp_i": qi})
        return out
    finally:
        _lib.kan_container_destroy(h)


def save_container(path: str, descriptor, coeffs, lut=None, spline_tables=None):
    """save_container (io.hpp:108-211): lut = dict(entries, k, h) or None;
    spline_tables = one dict per KAN layer (values, bits_a, h, qp_d, qp_i) or None."""
    text = descriptor if isinstance(descriptor, str) else json.dumps(descriptor)
    cs = [np.ascontiguousarray(c, dtype=np.float64) for c in coeffs]
    cp = (_vp * len(cs))(*[c.ctypes.data for c in cs])
    le = None if lut is None else np.ascontiguousarray(lut["entries"], dtype=np.uint8)
    sv = sp = sqd = sqi = None
    ba = hv = 0
    if spline_tables:
        vals = [np.ascontiguousarray(t["values"], dtype=np.uint8).ravel() for t in spline_tables]
        sv = (_vp * len(vals))(*[v.ctypes.data for v in vals])
        sqd = np.ascontiguousarray(np.stack([t["qp_d"] for t in spline_tables]), dtype=np.float64)
        sqi = np.ascontiguousarray(np.stack([t["qp_i"] for t in spline_tables]), dtype=np.int64)
        ba, hv = int(spline_tables[0]["bits_a"]), int(spline_tables[0]["h"])
        sp = vals
    st = _lib.kan_container_save(str(path).encode(), text.encode(), cp,
                                 None if le is None else le.ctypes.data,
                                 0 if le is None else le.size,
                                 0 if lut is None else int(lut["k"]), 0 if lut is None else int(lut["h"]),
                                 sv, ba, hv, None if sqd is None else sqd.ctypes.data,
                                 None if sqi is None else sqi.ctypes.data)
    del sp
    if st != KAN_OK:
        raise _STATUS.get(st, RuntimeError)(KanError(st, _lib.kan_container_save_error().decode()))


def eval_mode_from_string(s: str) -> int:
    """eval.hpp:19-25, plus the engine's bf16 datapath."""
    table = {"fp32": MODE_FP32, "bf16": MODE_BF16, "bspline-lut": MODE_BSPLINE_LUT,
             "spline-table": MODE_SPLINE_TABLE, "fake-quant": MODE_FAKE_QUANT}
    if s not in table:
        raise ValueError(f"unknown evaluation mode '{s}'")
    return table[s]


def build_bspline_lut(degree: int, k: int, h: int) -> np.ndarray:
    """build_bspline_lut (lut.hpp:103-131) through the engine's host code."""
    n = _lib.kan_lut_build(degree, k, h, None, 0)
    if n < 0:
        raise ValueError("build_bspline_lut: bad arguments")
    out = np.zeros(n, dtype=np.uint8)
    _lib.kan_lut_build(degree, k, h, out.ctypes.data, n)
    return out


@dataclass
class EvalOptions:
    """EvalOptions (eval.hpp:37-45) extended with the engine's choices.

    spline-table mode reads lut_k as the tables' input bits (bits_a) and lut_h as
    their value bits (h), as run_sweep passes (bits_a, bits_b) (sweep.hpp:247-253);
    fake-quant mode reads bits_w, lut_k = bits_a and lut_h = bits_b (32 = passthrough)."""
    mode: str = "fp32"
    lut_k: int = 8
    lut_h: int = 8
    bits_w: int = 8
    w_scheme: int = W_PER_CHANNEL_SYM
    silu_base: bool = False
    out_kind: int = OUT_F32
    out_scale: float = 1.0
    split_k: int = 0
    # fake-quant calibrated policy: one (lo, hi) per KAN layer (EvalOptions::a_ranges)
    a_ranges: Optional[Sequence] = None


def _torch():
    import torch  # plumbing only: device buffers and streams
    return torch


class Engine:
    """A configured model on one CUDA device (model_from_descriptor + PreparedModel)."""

    def __init__(self, descriptor, device: int = 0):
        text = descriptor if isinstance(descriptor, str) else json.dumps(descriptor)
        try:
            self.descriptor = json.loads(text)
        except ValueError:
            self.descriptor = None  # the C++ parser reports the format error
        h = _vp()
        st = _lib.kan_engine_create(text.encode(), device, C.byref(h))
        self._h = h
        if st != KAN_OK:
            msg = _lib.kan_engine_last_error(h).decode() if h else ""
            self.close()
            raise _STATUS.get(st, RuntimeError)(KanError(st, msg))
        self.device = device
        self.opts: Optional[EvalOptions] = None

    @classmethod
    def load(cls, path: str, device: int = 0) -> "Engine":
        """load_model (io.hpp:352) into an engine: the container's model,
        coefficients, spline tables and LUT."""
        self = cls.__new__(cls)
        h = _vp()
        st = _lib.kan_engine_load(str(path).encode(), device, C.byref(h))
        self._h = h
        if st != KAN_OK:
            msg = _lib.kan_engine_last_error(h).decode() if h else ""
            self.close()
            raise _STATUS.get(st, RuntimeError)(KanError(st, msg))
        self.descriptor = load_container(path)["descriptor"]
        self.device = device
        self.opts = None
        return self

    # -- lifetime ---------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            _lib.kan_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != KAN_OK:
            msg = _lib.kan_engine_last_error(self._h).decode()
            raise _STATUS.get(st, RuntimeError)(KanError(st, msg))

    # -- model shape ---------------------------------------------------------------
    @property
    def num_kan_layers(self) -> int:
        return _lib.kan_engine_num_kan_layers(self._h)

    @property
    def input_size(self) -> int:
        return _lib.kan_engine_input_size(self._h)

    @property
    def output_count(self) -> int:
        return _lib.kan_engine_output_count(self._h)

    def layer_shape(self, i):
        a, b = C.c_int(), C.c_int()
        self._check(_lib.kan_engine_layer_shape(self._h, i, C.byref(a), C.byref(b)))
        return a.value, b.value

    # -- weights / configuration -------------------------------------------------
    def set_coeffs(self, layer: int, coeffs, base_w=None):
        c = np.ascontiguousarray(coeffs, dtype=np.float64)
        b = None if base_w is None else np.ascontiguousarray(base_w, dtype=np.float64)
        self._check(_lib.kan_engine_set_coeffs(self._h, layer, c.ctypes.data, c.size,
                                               None if b is None else b.ctypes.data,
                                               0 if b is None else b.size))

    def configure(self, opts: EvalOptions):
        if opts.a_ranges is None:
            self._check(_lib.kan_engine_set_activation_ranges(self._h, None, 0))
        else:
            rg = np.ascontiguousarray(opts.a_ranges, dtype=np.float64).reshape(-1, 2)
            self._check(_lib.kan_engine_set_activation_ranges(self._h, rg.ctypes.data, rg.shape[0]))
        cfg = _Config(eval_mode_from_string(opts.mode), opts.lut_k, opts.lut_h, opts.bits_w,
                      opts.w_scheme, int(bool(opts.silu_base)), opts.out_kind,
                      float(opts.out_scale), opts.split_k)
        self._check(_lib.kan_engine_configure(self._h, C.byref(cfg)))
        self.opts = opts

    # -- forward paths -------------------------------------------------------------
    def _stream(self, stream):
        torch = _torch()
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        return C.c_void_p(s.cuda_stream)

    def model_forward(self, x, out=None, stream=None):
        """model_forward (eval.hpp:200-253) on a CUDA fp32 tensor [batch, input_size]."""
        torch = _torch()
        assert x.is_cuda and x.dtype == torch.float32 and x.is_contiguous()
        M = x.shape[0]
        i8 = self.opts is not None and self.opts.out_kind == OUT_I8
        if out is None:
            out = torch.empty((M, self.output_count), device=x.device,
                              dtype=torch.int8 if i8 else torch.float32)
        self._check(_lib.kan_engine_forward(self._h, x.data_ptr(), M, out.data_ptr(),
                                            self._stream(stream)))
        return out

    def forward_host(self, x: np.ndarray, stream=None) -> np.ndarray:
        """model_forward on host buffers: H2D and D2H are inside the call."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        i8 = self.opts is not None and self.opts.out_kind == OUT_I8
        out = np.empty((x.shape[0], self.output_count), dtype=np.int8 if i8 else np.float32)
        self._check(_lib.kan_engine_forward_host(self._h, x.ctypes.data, x.shape[0],
                                                 out.ctypes.data, self._stream(stream)))
        return out

    def forward_host_ptr(self, x_ptr: int, batch: int, out_ptr: int, stream=None):
        self._check(_lib.kan_engine_forward_host(self._h, x_ptr, batch, out_ptr,
                                                 self._stream(stream)))

    def predict(self, x, stream=None):
        """predict (eval.hpp:255-276): argmax of the logits, first maximum wins."""
        torch = _torch()
        labels = torch.empty(x.shape[0], device=x.device, dtype=torch.int32)
        self._check(_lib.kan_engine_predict(self._h, x.data_ptr(), x.shape[0],
                                            labels.data_ptr(), self._stream(stream)))
        return labels

    def evaluate_accuracy(self, x, labels, stream=None) -> float:
        """evaluate_accuracy (eval.hpp:279-287): top-1 accuracy against int32 labels."""
        torch = _torch()
        lab = labels.to(device=x.device, dtype=torch.int32).contiguous()
        acc = C.c_double()
        self._check(_lib.kan_engine_evaluate_accuracy(self._h, x.data_ptr(), lab.data_ptr(), x.shape[0],
                                                      C.byref(acc), self._stream(stream)))
        return acc.value

    # -- training (train.hpp) -----------------------------------------------------------
    def linear_backward(self, layer: int, x, dout, want_inputs: bool = True, stream=None):
        """kan_linear_backward (train.hpp:84-136) on CUDA fp32 tensors: (dcoeffs
        [n_in*(G+P), n_out], dinputs [batch, n_in] or None)."""
        torch = _torch()
        n_in, n_out = self.layer_shape(layer)
        nb = self.descriptor["grid"]["intervals"] + self.descriptor["grid"]["degree"]
        x = x.contiguous()
        dout = dout.contiguous()
        dc = torch.empty((n_in * nb, n_out), device=x.device, dtype=torch.float32)
        di = torch.empty((x.shape[0], n_in), device=x.device, dtype=torch.float32) if want_inputs else None
        self._check(_lib.kan_engine_linear_backward(self._h, layer, x.data_ptr(), x.shape[0], dout.data_ptr(),
                                                    dc.data_ptr(), None if di is None else di.data_ptr(),
                                                    self._stream(stream)))
        return dc, di

    def conv_backward(self, layer: int, x, dout, want_inputs: bool = True, stream=None):
        """The conv-layer backward of train() (train.hpp:367-399): x [batch, c_in, H, W]
        and dout [batch, c_out, Ho, Wo] as contiguous CUDA fp32 tensors (any 2-D view);
        returns (dcoeffs [c_in*K*K*(G+P), c_out], dinputs shaped like x or None)."""
        torch = _torch()
        n_in, n_out = self.layer_shape(layer)
        nb = self.descriptor["grid"]["intervals"] + self.descriptor["grid"]["degree"]
        x = x.contiguous()
        dout = dout.contiguous()
        dc = torch.empty((n_in * nb, n_out), device=x.device, dtype=torch.float32)
        di = torch.empty_like(x) if want_inputs else None
        self._check(_lib.kan_engine_conv_backward(self._h, layer, x.data_ptr(), x.shape[0], dout.data_ptr(),
                                                  dc.data_ptr(), None if di is None else di.data_ptr(),
                                                  self._stream(stream)))
        return dc, di

    def sgd_step(self, layer: int, dcoeffs, lr: float, momentum: float, stream=None):
        """One SGD-with-momentum update of a layer's coefficients on the device
        (train.hpp:361-366, 401-404): fp64 master copy and velocity stay resident,
        the fp32 copies the forward / backward read are refreshed in the same launch."""
        dcoeffs = dcoeffs.contiguous()
        self._check(_lib.kan_engine_sgd_step(self._h, layer, dcoeffs.data_ptr(), float(lr), float(momentum),
                                             self._stream(stream)))

    def get_coeffs(self, layer: int) -> np.ndarray:
        """The layer's current coefficients [n_in*(G+P), n_out] (after device-side updates)."""
        n_in, n_out = self.layer_shape(layer)
        nb = self.descriptor["grid"]["intervals"] + self.descriptor["grid"]["degree"]
        out = np.empty((n_in * nb, n_out), dtype=np.float64)
        self._check(_lib.kan_engine_get_coeffs(self._h, layer, out.ctypes.data, out.size))
        return out

    # -- parity probes ---------------------------------------------------------------
    def layer_levels(self, layer: int, x, stream=None):
        torch = _torch()
        out = torch.empty(x.shape, device=x.device, dtype=torch.int16)
        self._check(_lib.kan_engine_layer_levels(self._h, layer, x.data_ptr(), x.numel(),
                                                 out.data_ptr(), self._stream(stream)))
        return out.view(torch.uint16) if hasattr(torch, "uint16") else out

    def layer_accumulators(self, layer: int, levels, stream=None):
        torch = _torch()
        _, n_out = self.layer_shape(layer)
        M = levels.shape[0]
        acc_s = torch.zeros((M, n_out), device=levels.device, dtype=torch.int32)
        acc_b = torch.zeros((M, n_out), device=levels.device, dtype=torch.int32)
        self._check(_lib.kan_engine_layer_accumulators(self._h, layer, levels.data_ptr(), M,
                                                       acc_s.data_ptr(), acc_b.data_ptr(),
                                                       self._stream(stream)))
        return acc_s, acc_b

    def set_spline_tables(self, layer: int, tables):
        """Supply a layer's SplineTableSet (dict with values [n_in, n_out, 2^bits_a] u8,
        bits_a, h, qp_d = (in_scale, out_scale), qp_i = (in_zp, in_qhi, out_zp,
        out_qhi)) instead of building it from the coefficients; None clears."""
        if tables is None:
            self._check(_lib.kan_engine_set_spline_tables(self._h, layer, None, 0, 0, 0, None, None))
            return
        v = np.ascontiguousarray(tables["values"], dtype=np.uint8)
        qd = np.ascontiguousarray(tables["qp_d"], dtype=np.float64)
        qi = np.ascontiguousarray(tables["qp_i"], dtype=np.int64)
        self._check(_lib.kan_engine_set_spline_tables(self._h, layer, v.ctypes.data, v.size,
                                                      int(tables["bits_a"]), int(tables["h"]),
                                                      qd.ctypes.data, qi.ctypes.data))

    def spline_table(self, layer: int):
        """The configured SplineTableSet of one KAN layer (reference layout)."""
        qd = np.zeros(2)
        qi = np.zeros(4, dtype=np.int64)
        n = _lib.kan_engine_spline_table(self._h, layer, None, 0, qd.ctypes.data, qi.ctypes.data)
        if n < 0:
            self._check(int(-n))
        n_in, n_out = self.layer_shape(layer)
        out = np.zeros(n, dtype=np.uint8)
        n2 = _lib.kan_engine_spline_table(self._h, layer, out.ctypes.data, n, None, None)
        if n2 < 0:
            self._check(int(-n2))
        bits_a = int(n // (n_in * n_out)).bit_length() - 1 if n_in * n_out else 0
        return {"values": out.reshape(n_in, n_out, -1), "qp_d": qd, "qp_i": qi, "bits_a": bits_a,
                "h": int(qi[3] + 1).bit_length() - 1, "n_in": n_in, "n_out": n_out}

    def lut(self) -> np.ndarray:
        n = _lib.kan_engine_lut(self._h, None, 0)
        out = np.zeros(n, dtype=np.uint8)
        if n:
            _lib.kan_engine_lut(self._h, out.ctypes.data, n)
        return out

    @property
    def last_launches(self) -> int:
        return _lib.kan_engine_last_launches(self._h)

    def set_option(self, name: str, value: int):
        """kan_engine_set_option: a tuning / debug switch (OPTIONS); takes effect at
        the next configure (record_plan: at the next forward)."""
        self._check(_lib.kan_engine_set_option(self._h, OPTIONS[name], int(value)))

    @property
    def last_plan(self) -> str:
        """Launch plan of the last forward (needs set_option('record_plan', 1))."""
        return _lib.kan_engine_last_plan(self._h).decode()

    def set_profiling(self, on: bool):
        self._check(_lib.kan_engine_set_profiling(self._h, int(bool(on))))

    def layer_timeline(self, layer: int) -> np.ndarray:
        """[ctas, 8] %globaltimer stamps of the layer's last launch (option timeline=1)."""
        n = _lib.kan_engine_layer_timeline(self._h, layer, None, 0)
        out = np.zeros(max(n, 0), dtype=np.uint64)
        if n > 0:
            _lib.kan_engine_layer_timeline(self._h, layer, out.ctypes.data, n)
        return out.reshape(-1, 8)

    def layer_time_ms(self, layer: int):
        """(accumulated device ms, launches) of one KAN layer since profiling was enabled."""
        ms, n = C.c_double(), C.c_int64()
        self._check(_lib.kan_engine_layer_time_ms(self._h, layer, C.byref(ms), C.byref(n)))
        return ms.value, n.value


# ---- single-layer conveniences mirroring the reference's layer entry points ----

def _linear_descriptor(n_in, n_out, G, P, lo=-1.0, hi=1.0):
    return {"name": "layer", "grid": {"intervals": G, "degree": P}, "input": [n_in],
            "domain": [lo, hi], "layers": [{"type": "linear", "n_in": n_in, "n_out": n_out}]}


def tabulated_kan_forward(acts, coeffs, G: int, P: int, k: int, h: int, bits_w: int,
                          w_scheme: int = W_PER_TENSOR_ASYM, lo=-1.0, hi=1.0, device=0):
    """tabulated_kan_forward (lut.hpp:217-231) for one linear layer, on the GPU."""
    n_in, n_out = acts.shape[1], coeffs.shape[1]
    e = Engine(_linear_descriptor(n_in, n_out, G, P, lo, hi), device)
    e.set_coeffs(0, coeffs)
    e.configure(EvalOptions(mode="bspline-lut", lut_k=k, lut_h=h, bits_w=bits_w,
                            w_scheme=w_scheme))
    return e.model_forward(acts)


def kan_linear_forward(acts, coeffs, G: int, P: int, mode: str = "fp32", lo=-1.0, hi=1.0,
                       device=0):
    """kan_linear_forward (layers.hpp:118-121) on the fp32 or bf16 datapath."""
    n_in, n_out = acts.shape[1], coeffs.shape[1]
    e = Engine(_linear_descriptor(n_in, n_out, G, P, lo, hi), device)
    e.set_coeffs(0, coeffs)
    e.configure(EvalOptions(mode=mode))
    return e.model_forward(acts)


def build_spline_tables(coeffs, n_in: int, n_out: int, G: int, P: int, bits_a: int, h: int,
                        lo=-1.0, hi=1.0, device=0):
    """build_spline_tables (spline_table.hpp:87-95) for a linear layer, built on the GPU."""
    e = Engine(_linear_descriptor(n_in, n_out, G, P, lo, hi), device)
    e.set_coeffs(0, coeffs)
    e.configure(EvalOptions(mode="spline-table", lut_k=bits_a, lut_h=h))
    return e.spline_table(0)


def spline_table_forward(acts, tables, G: int = 5, P: int = 3, lo=-1.0, hi=1.0, device=0):
    """spline_table_forward (spline_table.hpp:90-107) over a SplineTableSet dict, on the GPU."""
    n_in, n_out = tables["n_in"], tables["n_out"]
    if acts.shape[1] != n_in:
        raise ValueError(f"spline_table_forward: shape mismatch: got {acts.shape[1]} inputs, "
                         f"tables expect {n_in}")
    e = Engine(_linear_descriptor(n_in, n_out, G, P, lo, hi), device)
    e.set_spline_tables(0, tables)
    e.configure(EvalOptions(mode="spline-table", lut_k=tables["bits_a"], lut_h=tables["h"]))
    return e.model_forward(acts)


def softmax_cross_entropy(logits, labels, stream=None):
    """softmax_cross_entropy (train.hpp:139-160) on the GPU: (mean loss, dlogits)."""
    torch = _torch()
    logits = logits.contiguous()
    lab = labels.to(device=logits.device, dtype=torch.int32).contiguous()
    M, n = logits.shape
    rows = torch.empty(M, device=logits.device, dtype=torch.float32)
    d = torch.empty_like(logits)
    s = stream if stream is not None else torch.cuda.current_stream(logits.device)
    st = _lib.kan_softmax_cross_entropy(logits.data_ptr(), lab.data_ptr(), M, n, rows.data_ptr(), d.data_ptr(),
                                        C.c_void_p(s.cuda_stream))
    if st != KAN_OK:
        raise _STATUS.get(st, RuntimeError)(KanError(st, "softmax_cross_entropy"))
    return float(rows.double().mean().item()) if M else 0.0, d


def maxpool2(x, channels: int, H: int, W: int, window: int = 2, stream=None):
    """maxpool2 (layers.hpp:193-205) on NCHW fp32 rows [batch, C*H*W] -> [batch, C*Ho*Wo]."""
    torch = _torch()
    x = x.contiguous()
    M = x.shape[0]
    out = torch.empty((M, channels * (H // window) * (W // window)), device=x.device, dtype=torch.float32)
    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    st = _lib.kan_maxpool2_f32(x.data_ptr(), M * channels, H, W, window, out.data_ptr(), C.c_void_p(s.cuda_stream))
    if st != KAN_OK:
        raise _STATUS.get(st, RuntimeError)(KanError(st, "maxpool2"))
    return out


def maxpool2_backward(x, dout, channels: int, H: int, W: int, window: int = 2, stream=None):
    """The pooling backward of train() (train.hpp:407-431)."""
    torch = _torch()
    x = x.contiguous()
    dout = dout.contiguous()
    din = torch.empty_like(x)
    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    st = _lib.kan_maxpool2_backward_f32(x.data_ptr(), x.shape[0] * channels, H, W, window, dout.data_ptr(),
                                        din.data_ptr(), C.c_void_p(s.cuda_stream))
    if st != KAN_OK:
        raise _STATUS.get(st, RuntimeError)(KanError(st, "maxpool2_backward"))
    return din

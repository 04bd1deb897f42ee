"""ctypes bindings for the CPU checkers (TEST INFRASTRUCTURE ONLY).

- ``Oracle``: the C restatement in ``oracle/kan_oracle.c`` (always present
  once ``make -C oracle`` or ``__graft_entry__.build()`` ran).
- ``Ref``: the unmodified reference headers compiled into
  ``oracle/_ref/libkantize_ref.so`` (present where /root/reference was
  available at build time; the .so travels with the repo snapshot).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libkan_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libkantize_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_fp = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(dtype=np.uint16, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class _Grid(C.Structure):
    _fields_ = [("intervals", C.c_int), ("degree", C.c_int), ("lo", C.c_double),
                ("hi", C.c_double), ("delta", C.c_double)]


class _IntLayer(C.Structure):
    _fields_ = [("wscheme", C.c_int), ("bits_w", C.c_int), ("silu", C.c_int),
                ("qw_u8", C.c_void_p), ("s_w", C.c_double), ("z_w", C.c_int64),
                ("qw_s8", C.c_void_p), ("s_wc", C.c_void_p),
                ("silu_codes", C.c_void_p), ("s_s", C.c_double), ("z_s", C.c_int64),
                ("qwb", C.c_void_p), ("s_wb", C.c_void_p)]


class Oracle:
    """The C restatement of the reference hot path (kan_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_oracle()
        L = self.lib = C.CDLL(path)
        G = C.POINTER(_Grid)
        L.kor_grid_build.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, G]
        L.kor_clamp.argtypes = [G, C.c_double]
        L.kor_clamp.restype = C.c_double
        L.kor_basis_at_coord.argtypes = [G, C.c_double, _dp]
        L.kor_knot_coord.argtypes = [G, C.c_double]
        L.kor_knot_coord.restype = C.c_double
        L.kor_quant_params.argtypes = [C.c_double, C.c_double, C.c_int, C.POINTER(C.c_double),
                                       C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.kor_quantize.argtypes = [C.c_double, C.c_double, C.c_int64, C.c_int64, C.c_int64]
        L.kor_quantize.restype = C.c_int64
        L.kor_level_of.argtypes = [G, C.c_int, C.c_double]
        L.kor_level_of.restype = C.c_int64
        L.kor_levels_f32.argtypes = [G, C.c_int, _fp, C.c_size_t, _u16p]
        L.kor_levels_f64.argtypes = [G, C.c_int, _dp, C.c_size_t, _u16p]
        L.kor_lut_size.argtypes = [C.c_int, C.c_int]
        L.kor_lut_size.restype = C.c_size_t
        L.kor_build_lut.argtypes = [C.c_int, C.c_int, C.c_int, _u8p, C.c_size_t]
        L.kor_lut_lookup.argtypes = [G, C.c_int, _u8p, C.c_int64, _u8p, C.POINTER(C.c_int)]
        L.kor_quantized_basis_reference.argtypes = [G, C.c_int, C.c_int, C.c_int64, _u8p,
                                                    C.POINTER(C.c_int)]
        L.kor_linear_forward_fp64.argtypes = [G, C.c_int64, C.c_int, C.c_int, _dp, _dp, _dp]
        L.kor_lut_forward_fp64.argtypes = [G, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int,
                                           C.c_int, _dp, _dp, _dp]
        L.kor_wquant_per_tensor.argtypes = [_dp, C.c_size_t, C.c_int, _u8p,
                                            C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        L.kor_wquant_per_channel_sym.argtypes = [_dp, C.c_int64, C.c_int, C.c_int, _i8p, _dp]
        L.kor_wquant_joint.argtypes = [_dp, _dp, C.c_int64, C.c_int, C.c_int, C.c_int,
                                       C.c_double, _i8p, _i8p, _dp]
        L.kor_silu_table.argtypes = [G, C.c_int, _u8p, C.POINTER(C.c_double),
                                     C.POINTER(C.c_int64)]
        L.kor_int_accumulate.argtypes = [G, C.c_int, _u8p, C.POINTER(_IntLayer), C.c_int64,
                                         C.c_int, C.c_int, _u16p, _i32p, _i32p, _i64p]
        L.kor_int_layer_forward.argtypes = [G, C.c_int, C.c_int, _u8p, C.POINTER(_IntLayer),
                                            C.c_int64, C.c_int, C.c_int, _u16p, _dp]
        L.kor_requant_i8.argtypes = [C.c_double, C.c_double]
        L.kor_requant_i8.restype = C.c_int8
        L.kor_im2col.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        L.kor_fakequant_forward_fp64.argtypes = [G, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int,
                                                 C.c_int, _dp, _dp, _dp]
        L.kor_spline_tables_build.argtypes = [G, _dp, C.c_int, C.c_int, C.c_int, C.c_int, _u8p,
                                              _dp, _i64p]
        L.kor_spline_level.argtypes = [C.c_double, C.c_double, C.c_int64, C.c_int64]
        L.kor_spline_level.restype = C.c_int64
        L.kor_spline_table_accumulate.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int64,
                                                  C.c_int64, _u8p, _i64p]
        L.kor_spline_table_forward.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, _dp, _i64p,
                                               C.c_int64, _dp, _dp]

    # -- grid / quant ---------------------------------------------------------
    def grid(self, G, P, lo=-1.0, hi=1.0):
        g = _Grid()
        if self.lib.kor_grid_build(G, P, lo, hi, C.byref(g)):
            raise ValueError("build_grid: bad arguments")
        return g

    def quant_params(self, a, b, bits):
        s, z, qh = C.c_double(), C.c_int64(), C.c_int64()
        if self.lib.kor_quant_params(a, b, bits, C.byref(s), C.byref(z), C.byref(qh)):
            raise ValueError("compute_quant_params: bad arguments")
        return s.value, z.value, qh.value

    def basis(self, g, x):
        nb = g.intervals + g.degree
        out = np.zeros(nb)
        xi = self.lib.kor_knot_coord(C.byref(g), x)
        start = self.lib.kor_basis_at_coord(C.byref(g), xi, out)
        return out, start

    def level_of(self, g, k, x):
        return self.lib.kor_level_of(C.byref(g), k, float(x))

    def levels(self, g, k, x):
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty(x.shape, dtype=np.uint16)
        self.lib.kor_levels_f32(C.byref(g), k, x.ravel(), x.size, out.ravel())
        return out

    def lut(self, P, k, h):
        n = self.lib.kor_lut_size(P, k)
        out = np.zeros(n, dtype=np.uint8)
        if self.lib.kor_build_lut(P, k, h, out, n) < 0:
            raise ValueError("build_bspline_lut: bad arguments")
        return out

    def lut_lookup(self, g, k, lut, a):
        vals = np.zeros(16, dtype=np.uint8)
        start = C.c_int()
        cnt = self.lib.kor_lut_lookup(C.byref(g), k, lut, a, vals, C.byref(start))
        if cnt < 0:
            raise IndexError("lut_basis_lookup: lattice level out of range")
        return vals[:cnt].copy(), start.value

    def quantized_basis_reference(self, g, k, h, a):
        vals = np.zeros(16, dtype=np.uint8)
        start = C.c_int()
        cnt = self.lib.kor_quantized_basis_reference(C.byref(g), k, h, a, vals, C.byref(start))
        return vals[:cnt].copy(), start.value

    # -- forwards -----------------------------------------------------------
    def linear_forward(self, g, acts, coeffs):
        acts = np.ascontiguousarray(acts, dtype=np.float64)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        M, n_in = acts.shape
        n_out = coeffs.shape[1]
        out = np.zeros((M, n_out))
        self.lib.kor_linear_forward_fp64(C.byref(g), M, n_in, n_out, acts, coeffs, out)
        return out

    def lut_forward(self, g, k, h, bits_w, acts, coeffs):
        acts = np.ascontiguousarray(acts, dtype=np.float64)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        M, n_in = acts.shape
        n_out = coeffs.shape[1]
        out = np.zeros((M, n_out))
        if self.lib.kor_lut_forward_fp64(C.byref(g), k, h, bits_w, M, n_in, n_out, acts,
                                         coeffs, out):
            raise ValueError("tabulated_kan_forward failed")
        return out

    def wquant_per_tensor(self, w, bits):
        w = np.ascontiguousarray(w, dtype=np.float64)
        q = np.zeros(w.shape, dtype=np.uint8)
        s, z = C.c_double(), C.c_int64()
        if self.lib.kor_wquant_per_tensor(w.ravel(), w.size, bits, q.ravel(), C.byref(s),
                                          C.byref(z)):
            raise ValueError("per-tensor quantization failed")
        return q, s.value, z.value

    def wquant_per_channel(self, w, bits):
        w = np.ascontiguousarray(w, dtype=np.float64)
        K, N = w.shape
        q = np.zeros((K, N), dtype=np.int8)
        s = np.zeros(N)
        if self.lib.kor_wquant_per_channel_sym(w, K, N, bits, q, s):
            raise ValueError("per-channel quantization failed")
        return q, s

    def silu_table(self, g, k):
        L = (g.intervals << k) + 1
        codes = np.zeros(L, dtype=np.uint8)
        s, z = C.c_double(), C.c_int64()
        self.lib.kor_silu_table(C.byref(g), k, codes, C.byref(s), C.byref(z))
        return codes, s.value, z.value

    def int_layer(self, g, k, h, wscheme, bits_w, coeffs, base_w=None):
        """Quantize one layer's weights the way the engine's LUT path does."""
        d = {"wscheme": wscheme, "bits_w": bits_w, "silu": base_w is not None,
             "lut": self.lut(g.degree, k, h)}
        if wscheme == 0:
            d["qw_u8"], d["s_w"], d["z_w"] = self.wquant_per_tensor(coeffs, bits_w)
        elif base_w is None:
            d["qw_s8"], d["s_wc"] = self.wquant_per_channel(coeffs, bits_w)
        if base_w is not None:
            d["silu_codes"], d["s_s"], d["z_s"] = self.silu_table(g, k)
            s_b = 1.0 / ((1 << h) - 1)
            d["qw_s8"], d["qwb"], d["s_wc"] = self.wquant_joint(coeffs, base_w, bits_w,
                                                                d["s_s"] / s_b)
            d["s_wb"] = np.zeros(coeffs.shape[1])
        return d

    def wquant_joint(self, w, wb, bits, ratio):
        w = np.ascontiguousarray(w, dtype=np.float64)
        wb = np.ascontiguousarray(wb, dtype=np.float64)
        K, N = w.shape
        q = np.zeros((K, N), dtype=np.int8)
        qb = np.zeros(wb.shape, dtype=np.int8)
        s = np.zeros(N)
        if self.lib.kor_wquant_joint(w, wb, K, wb.shape[0], N, bits, ratio, q, qb, s):
            raise ValueError("joint quantization failed")
        return q, qb, s

    def _int_struct(self, d):
        s = _IntLayer()
        s.wscheme, s.bits_w, s.silu = d["wscheme"], d["bits_w"], int(bool(d["silu"]))
        keep = []

        def ptr(a):
            keep.append(a)
            return a.ctypes.data

        if d["wscheme"] == 0:
            s.qw_u8, s.s_w, s.z_w = ptr(d["qw_u8"]), d["s_w"], d["z_w"]
        else:
            s.qw_s8, s.s_wc = ptr(d["qw_s8"]), ptr(d["s_wc"])
        if d["silu"]:
            s.silu_codes, s.s_s, s.z_s = ptr(d["silu_codes"]), d["s_s"], d["z_s"]
            s.qwb, s.s_wb = ptr(d["qwb"]), ptr(d["s_wb"])
        return s, keep

    def int_accumulate(self, g, k, d, levels, n_out):
        levels = np.ascontiguousarray(levels, dtype=np.uint16)
        M, n_in = levels.shape
        s, keep = self._int_struct(d)
        acc_s = np.zeros((M, n_out), dtype=np.int32)
        acc_b = np.zeros((M, n_out), dtype=np.int32)
        rs = np.zeros(max(M, 1), dtype=np.int64)
        if self.lib.kor_int_accumulate(C.byref(g), k, d["lut"], C.byref(s), M, n_in, n_out,
                                       levels, acc_s, acc_b, rs):
            raise ValueError("int accumulate failed")
        return acc_s, acc_b, rs[:M]

    def int_layer_forward(self, g, k, h, d, levels, n_out):
        levels = np.ascontiguousarray(levels, dtype=np.uint16)
        M, n_in = levels.shape
        s, keep = self._int_struct(d)
        y = np.zeros((M, n_out))
        if self.lib.kor_int_layer_forward(C.byref(g), k, h, d["lut"], C.byref(s), M, n_in,
                                          n_out, levels, y):
            raise ValueError("int layer forward failed")
        return y

    def requant_i8(self, y, s_out):
        f = np.vectorize(lambda v: self.lib.kor_requant_i8(float(v), s_out), otypes=[np.int8])
        return f(y)

    def im2col(self, x, kernel, stride, padding):
        x = np.ascontiguousarray(x, dtype=np.float64)
        Cc, H, W = x.shape
        Ho = (H + 2 * padding - kernel) // stride + 1
        Wo = (W + 2 * padding - kernel) // stride + 1
        out = np.zeros((Ho * Wo, kernel * kernel * Cc))
        if self.lib.kor_im2col(x, Cc, H, W, kernel, stride, padding, out):
            raise ValueError("im2col: output dimensions are not positive integers")
        return out


    def levels_f64(self, g, k, y):
        """Next-layer lattice levels of fp64 layer outputs (clamp + quantize)."""
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = np.zeros(y.shape, dtype=np.uint16)
        self.lib.kor_levels_f64(C.byref(g), k, y.ravel(), y.size, out.ravel())
        return out

    @staticmethod
    def im2col_levels(lv, kernel, stride, padding, pad_level):
        """im2col (layers.hpp:126-154) over lattice levels [M, C, H, W] ->
        [M*Ho*Wo, C*K*K] in the reference's channel-major column order.  Padded
        taps hold level(0.0) (the reference leaves them 0.0 and the basis is
        evaluated there).  Output size uses floor semantics; with a stride that
        does not divide the padded span this equals the reference on the input
        zero-extended at the bottom/right (stride-2 recipe)."""
        M, Cc, H, W = lv.shape
        Ho = (H + 2 * padding - kernel) // stride + 1
        Wo = (W + 2 * padding - kernel) // stride + 1
        ph = max(H + 2 * padding, stride * (Ho - 1) + kernel)
        pw = max(W + 2 * padding, stride * (Wo - 1) + kernel)
        pad = np.full((M, Cc, ph, pw), pad_level, dtype=np.uint16)
        pad[:, :, padding:padding + H, padding:padding + W] = lv
        taps = []
        for ky in range(kernel):
            for kx in range(kernel):
                taps.append(pad[:, :, ky:ky + stride * (Ho - 1) + 1:stride,
                                kx:kx + stride * (Wo - 1) + 1:stride])
        t = np.stack(taps, axis=2)  # [M, C, KK, Ho, Wo]
        return np.ascontiguousarray(t.transpose(0, 3, 4, 1, 2)).reshape(M * Ho * Wo,
                                                                        Cc * kernel * kernel)

    # -- fake-quant mode (eval.hpp:106-159) ----------------------------------------
    def fakequant_forward(self, g, bits_w, bits_a, bits_b, acts, coeffs):
        acts = np.ascontiguousarray(acts, dtype=np.float64)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        out = np.zeros((acts.shape[0], coeffs.shape[1]))
        if self.lib.kor_fakequant_forward_fp64(C.byref(g), bits_w, bits_a, bits_b, acts.shape[0],
                                               acts.shape[1], coeffs.shape[1], acts, coeffs, out):
            raise ValueError("fake-quant: bad arguments")
        return out

    def fakequant_model_forward(self, desc, Ws, x, bits_w, bits_a, bits_b):
        """model_forward in fake-quant mode over linear / conv / maxpool / flatten
        (conv: im2col of the fake-quantized input, padded taps 0.0)."""
        G, P = desc["grid"]["intervals"], desc["grid"]["degree"]
        lo, hi = desc.get("domain", [-1.0, 1.0])
        g = self.grid(G, P, lo, hi)
        M = x.shape[0]
        v = np.asarray(x, dtype=np.float64).reshape(M, *desc["input"])
        ki = 0
        for l in desc["layers"]:
            typ = l["type"]
            if typ == "linear":
                v = self.fakequant_forward(g, bits_w, bits_a, bits_b, v.reshape(M, -1), Ws[ki])
                ki += 1
            elif typ == "conv":
                kk, s_, p_ = l["kernel"], l.get("stride", 1), l.get("padding", 0)
                Ho = (v.shape[2] + 2 * p_ - kk) // s_ + 1
                Wo = (v.shape[3] + 2 * p_ - kk) // s_ + 1
                vq = v
                if bits_a != 32:  # forward_conv fake-quantizes the tensor, then im2col pads 0.0
                    s, z, qh = self.quant_params(lo, hi, bits_a)
                    vq = s * (np.clip(np.vectorize(lambda t: self.lib.kor_quantize(float(t), s, z, 0, qh),
                                                   otypes=[np.int64])(v), 0, qh) - z)
                cols = np.concatenate([self.im2col(vq[m], kk, s_, p_) for m in range(M)])
                y = self.fakequant_forward(g, bits_w, 32, bits_b, cols, Ws[ki])
                v = y.reshape(M, Ho, Wo, -1).transpose(0, 3, 1, 2)
                ki += 1
            elif typ == "maxpool":
                w = l.get("window", 2)
                Ho, Wo = v.shape[2] // w, v.shape[3] // w
                v = v[:, :, :Ho * w, :Wo * w].reshape(M, v.shape[1], Ho, w, Wo, w).max(axis=(3, 5))
            elif typ == "flatten":
                v = v.reshape(M, -1)
        return v

    # -- spline-table mode (spline_table.hpp) ------------------------------------
    def spline_tables(self, g, coeffs, n_in, n_out, bits_a, h):
        """build_spline_tables: dict(values [n_in, n_out, 2^bits_a] u8, qp_d, qp_i)."""
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        vals = np.zeros(n_in * n_out << bits_a, dtype=np.uint8)
        qd, qi = np.zeros(2), np.zeros(4, dtype=np.int64)
        if self.lib.kor_spline_tables_build(C.byref(g), coeffs.ravel(), n_in, n_out, bits_a, h,
                                            vals, qd, qi):
            raise ValueError("build_spline_tables: invalid arguments")
        return {"values": vals.reshape(n_in, n_out, 1 << bits_a), "qp_d": qd, "qp_i": qi,
                "bits_a": bits_a, "h": h, "n_in": n_in, "n_out": n_out}

    def spline_levels(self, t, x):
        """quantize_value(x, in_qp) per element (u8)."""
        x = np.asarray(x, dtype=np.float64)
        s, z, qh = t["qp_d"][0], int(t["qp_i"][0]), int(t["qp_i"][1])
        f = np.vectorize(lambda v: self.lib.kor_spline_level(float(v), s, z, qh), otypes=[np.uint8])
        return f(x) if x.size else x.astype(np.uint8)

    def spline_accumulate(self, t, levels):
        lv = np.ascontiguousarray(levels, dtype=np.uint8)
        M = lv.shape[0]
        acc = np.zeros((M, t["n_out"]), dtype=np.int64)
        self.lib.kor_spline_table_accumulate(np.ascontiguousarray(t["values"]).ravel(), t["n_in"],
                                             t["n_out"], t["bits_a"], int(t["qp_i"][2]), M,
                                             lv.ravel(), acc)
        return acc

    def spline_forward(self, t, acts):
        acts = np.ascontiguousarray(acts, dtype=np.float64)
        out = np.zeros((acts.shape[0], t["n_out"]))
        self.lib.kor_spline_table_forward(np.ascontiguousarray(t["values"]).ravel(), t["n_in"],
                                          t["n_out"], t["bits_a"], t["qp_d"], t["qp_i"],
                                          acts.shape[0], acts, out)
        return out

    def spline_model_tables(self, desc, Ws, bits_a, h):
        G, P = desc["grid"]["intervals"], desc["grid"]["degree"]
        lo, hi = desc.get("domain", [-1.0, 1.0])
        g = self.grid(G, P, lo, hi)
        tabs, ki, shape = [], 0, list(desc["input"])
        for l in desc["layers"]:
            if l["type"] == "linear":
                tabs.append(self.spline_tables(g, Ws[ki], l["n_in"], l["n_out"], bits_a, h))
                ki += 1
            elif l["type"] == "conv":
                kk = l["kernel"]
                tabs.append(self.spline_tables(g, Ws[ki], l["c_in"] * kk * kk, l["c_out"], bits_a, h))
                ki += 1
        return tabs

    def spline_model_forward(self, desc, tabs, x):
        """model_forward in spline-table mode (eval.hpp:135-193, 200-253): fp64
        values flow between layers; each KAN layer quantizes its input with
        quantize_value and sums table entries; conv layers go through im2col
        (layers.hpp:126-154); maxpool2 / flatten act on values."""
        M = x.shape[0]
        v = np.asarray(x, dtype=np.float64).reshape(M, *desc["input"])
        ki = 0
        for l in desc["layers"]:
            typ = l["type"]
            if typ == "linear":
                v = self.spline_forward(tabs[ki], v.reshape(M, -1))
                ki += 1
            elif typ == "conv":
                kk, s_, p_ = l["kernel"], l.get("stride", 1), l.get("padding", 0)
                Ho = (v.shape[2] + 2 * p_ - kk) // s_ + 1
                Wo = (v.shape[3] + 2 * p_ - kk) // s_ + 1
                cols = np.concatenate([self.im2col(v[m], kk, s_, p_) for m in range(M)])
                y = self.spline_forward(tabs[ki], cols)
                v = y.reshape(M, Ho, Wo, -1).transpose(0, 3, 1, 2)
                ki += 1
            elif typ == "maxpool":
                w = l.get("window", 2)
                Ho, Wo = v.shape[2] // w, v.shape[3] // w
                v = v[:, :, :Ho * w, :Wo * w].reshape(M, v.shape[1], Ho, w, Wo, w).max(axis=(3, 5))
            elif typ == "flatten":
                v = v.reshape(M, -1)
            else:
                raise ValueError(typ)
        return v

    @staticmethod
    def storage_kinds(desc):
        """Engine storage rule (kan_engine.cpp plan_buffers): a stored tensor keeps
        fp32 values when a consumer needs values (residual add, average pool;
        passed back through maxpool / flatten views), else lattice levels.
        Returns (per-layer flags, flag for the model input)."""
        layers = desc["layers"]
        named, src = {"input": -1}, []
        for i, l in enumerate(layers):
            src.append(named[l["input_from"]] if "input_from" in l else i - 1)
            if "id" in l:
                named[l["id"]] = i
        need = [False] * len(layers)
        need_in = [False]

        def mark(t):
            if t >= 0:
                need[t] = True
            else:
                need_in[0] = True
        for i in range(len(layers) - 1, -1, -1):
            l = layers[i]
            if "residual" in l:
                mark(named[l["residual"]])
            if l["type"] == "global_avgpool":
                mark(src[i])
            if l["type"] in ("maxpool", "flatten") and need[i]:
                mark(src[i])
        return need, need_in[0]

    def int_model_forward(self, desc, Ws, Bs, x, k, h, wscheme, bits_w):
        """The engine's integer LUT path over a model descriptor, layer by layer:
        levels -> (im2col) -> integer layer -> fp64 epilogue (+ residual) ->
        stored as next-layer levels, or as fp32 values where a consumer needs
        values (storage_kinds); returns the last layer's fp64 output ([M, N] for
        linear, [M, C, Ho, Wo] for conv)."""
        G, P = desc["grid"]["intervals"], desc["grid"]["degree"]
        lo, hi = desc.get("domain", [-1.0, 1.0])
        g = self.grid(G, P, lo, hi)
        lvl0 = self.level_of(g, k, 0.0)
        need, need_in = self.storage_kinds(desc)
        M = x.shape[0]
        x = np.ascontiguousarray(x, np.float32).reshape(M, *desc["input"])
        tens = {-1: ("f32", x) if (need_in or len(desc["input"]) == 1)
                else ("lv", self.levels(g, k, x))}
        named = {"input": -1}

        def levels(t):
            return self.levels(g, k, t[1]) if t[0] == "f32" else t[1]
        ki = 0
        y = None
        layers = desc["layers"]
        for i, l in enumerate(layers):
            src = named[l["input_from"]] if "input_from" in l else i - 1
            t = tens[src]
            typ = l["type"]
            last = i + 1 == len(layers)
            if typ in ("conv", "linear"):
                d = self.int_layer(g, k, h, wscheme, bits_w, Ws[ki], Bs[ki])
                N = Ws[ki].shape[1]
                ki += 1
                lv = levels(t)
                if typ == "conv":
                    kk, s_, p_ = l["kernel"], l.get("stride", 1), l.get("padding", 0)
                    Ho = (lv.shape[2] + 2 * p_ - kk) // s_ + 1
                    Wo = (lv.shape[3] + 2 * p_ - kk) // s_ + 1
                    cols = self.im2col_levels(lv, kk, s_, p_, lvl0)
                    y = self.int_layer_forward(g, k, h, d, cols, N)
                    y = y.reshape(M, Ho, Wo, N).transpose(0, 3, 1, 2)
                else:
                    y = self.int_layer_forward(g, k, h, d, lv.reshape(M, -1), N)
                if "residual" in l:
                    r = tens[named[l["residual"]]]
                    assert r[0] == "f32"
                    y = y + r[1].astype(np.float64)
                if last:
                    return y
                tens[i] = ("f32", y.astype(np.float32)) if need[i] else ("lv", self.levels_f64(g, k, y))
            elif typ == "maxpool":
                w = l.get("window", 2)
                a = t[1]
                Ho, Wo = a.shape[2] // w, a.shape[3] // w
                v = a[:, :, :Ho * w, :Wo * w].reshape(M, a.shape[1], Ho, w, Wo, w)
                tens[i] = (t[0], v.max(axis=(3, 5)))
            elif typ == "global_avgpool":
                assert t[0] == "f32"
                v = t[1].reshape(M, t[1].shape[1], -1)
                acc = np.zeros(v.shape[:2])
                for q in range(v.shape[2]):  # position order, one rounding per add
                    acc = acc + v[:, :, q].astype(np.float64)
                tens[i] = ("f32", (acc / v.shape[2]).astype(np.float32))
            elif typ == "flatten":
                tens[i] = (t[0], t[1].reshape(M, -1))
            else:
                raise ValueError(typ)
            if "id" in l:
                named[l["id"]] = i
        return y


class Ref:
    """The unmodified reference headers behind oracle/ref_shim.cpp."""

    available = os.path.exists(REF_SO)

    def __init__(self, path: str = REF_SO):
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_quant_params.argtypes = [C.c_double, C.c_double, C.c_int, C.POINTER(C.c_double),
                                       C.POINTER(C.c_int64)]
        L.ref_quantize_value.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int]
        L.ref_quantize_value.restype = C.c_int64
        L.ref_level_of.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                   C.c_double]
        L.ref_level_of.restype = C.c_int64
        L.ref_levels_f32.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _fp,
                                     C.c_int64, _u16p]
        L.ref_clamp.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double]
        L.ref_clamp.restype = C.c_double
        L.ref_build_lut.argtypes = [C.c_int, C.c_int, C.c_int, _u8p, C.c_int64,
                                    C.POINTER(C.c_int64)]
        L.ref_lut_lookup.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                     C.c_int64, _u8p, C.POINTER(C.c_int)]
        L.ref_quantized_basis.argtypes = L.ref_lut_lookup.argtypes
        L.ref_cox_de_boor.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, _dp]
        L.ref_linear_forward.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int64,
                                         C.c_int, C.c_int, _dp, _dp, _dp]
        L.ref_lut_forward.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                      C.c_int, C.c_int64, C.c_int, C.c_int, _dp, _dp, _dp]
        L.ref_latticequant_forward.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double,
                                               C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int,
                                               _dp, _dp, _dp]
        L.ref_im2col.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        L.ref_conv_forward.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                       C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]
        L.ref_validate_descriptor.argtypes = [C.c_char_p]
        L.ref_graph_forward.argtypes = [C.c_char_p, C.POINTER(C.c_void_p), C.c_int, C.c_int,
                                        C.c_int, C.c_int64, _dp, C.c_int64, _dp, C.c_int]
        L.ref_spline_tables.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                        C.c_int, C.c_int, C.c_int, _dp, C.c_int, C.c_int, _u8p,
                                        C.c_int64, _dp, _i64p]
        L.ref_spline_tables.restype = C.c_int64
        L.ref_spline_table_forward.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _u8p, _dp, _i64p,
                                               C.c_int64, _dp, _dp]
        L.ref_st_model_forward.argtypes = [C.c_char_p, C.POINTER(C.c_void_p), C.c_int, C.c_int,
                                           C.c_int64, C.c_int64, _dp, C.c_int64, _dp, C.c_int,
                                           C.c_int64, C.c_int, C.POINTER(C.c_double)]
        L.ref_save_container.argtypes = [C.c_char_p, C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int,
                                         C.c_int, C.c_char_p]
        L.ref_load_container.argtypes = [C.c_char_p]
        L.ref_calibrate_ranges.argtypes = [C.c_char_p, C.POINTER(C.c_void_p), C.c_int64, C.c_int64, _dp, _dp]
        L.ref_fakequant_calibrated_forward.argtypes = [C.c_char_p, C.POINTER(C.c_void_p), C.c_int, C.c_int,
                                                       C.c_int, _dp, C.c_int64, C.c_int64, _dp, C.c_int64, _dp]
        L.ref_linear_backward.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int64, C.c_int,
                                          C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.ref_train.argtypes = [C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_int64, C.c_int64,
                                _dp, _i32p, C.c_double, C.c_double, C.c_int, C.c_int, C.c_uint64,
                                C.POINTER(C.c_double)]
        L.ref_softmax_ce.argtypes = [C.c_int64, C.c_int, _dp, _i32p, _dp, C.POINTER(C.c_double)]
        L.ref_model_forward.argtypes = [C.c_char_p, C.POINTER(C.c_void_p), C.c_int, C.c_int,
                                        C.c_int, C.c_int, C.c_int64, C.c_int64, _dp, C.c_int64,
                                        _dp, C.c_int, C.c_int64]

    def err(self):
        return self.lib.ref_last_error().decode()

    def quant_params(self, a, b, bits):
        s, z = C.c_double(), C.c_int64()
        if self.lib.ref_quant_params(a, b, bits, C.byref(s), C.byref(z)):
            raise ValueError(self.err())
        return s.value, z.value

    def level_of(self, G, P, k, x, lo=-1.0, hi=1.0):
        return self.lib.ref_level_of(G, P, lo, hi, k, float(x))

    def levels(self, G, P, k, x, lo=-1.0, hi=1.0):
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty(x.shape, dtype=np.uint16)
        self.lib.ref_levels_f32(G, P, lo, hi, k, x.ravel(), x.size, out.ravel())
        return out

    def lut(self, P, k, h):
        buf = np.zeros(4096, dtype=np.uint8)
        mb = C.c_int64()
        n = self.lib.ref_build_lut(P, k, h, buf, buf.size, C.byref(mb))
        if n < 0:
            raise ValueError(self.err())
        return buf[:n].copy(), mb.value

    def lut_lookup(self, G, P, k, h, a, lo=-1.0, hi=1.0):
        vals = np.zeros(16, dtype=np.uint8)
        st = C.c_int()
        n = self.lib.ref_lut_lookup(G, P, lo, hi, k, h, a, vals, C.byref(st))
        if n < 0:
            raise IndexError(self.err())
        return vals[:n].copy(), st.value

    def quantized_basis(self, G, P, k, h, a, lo=-1.0, hi=1.0):
        vals = np.zeros(16, dtype=np.uint8)
        st = C.c_int()
        n = self.lib.ref_quantized_basis(G, P, lo, hi, k, h, a, vals, C.byref(st))
        return vals[:n].copy(), st.value

    def cox_de_boor(self, G, P, x, lo=-1.0, hi=1.0):
        out = np.zeros(G + P)
        st = self.lib.ref_cox_de_boor(G, P, lo, hi, x, out)
        return out, st

    def linear_forward(self, G, P, acts, coeffs, lo=-1.0, hi=1.0):
        acts = np.ascontiguousarray(acts, dtype=np.float64)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        out = np.zeros((acts.shape[0], coeffs.shape[1]))
        if self.lib.ref_linear_forward(G, P, lo, hi, acts.shape[0], acts.shape[1],
                                       coeffs.shape[1], acts, coeffs, out):
            raise ValueError(self.err())
        return out

    def lut_forward(self, G, P, k, h, bits_w, acts, coeffs, lo=-1.0, hi=1.0):
        acts = np.ascontiguousarray(acts, dtype=np.float64)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        out = np.zeros((acts.shape[0], coeffs.shape[1]))
        if self.lib.ref_lut_forward(G, P, lo, hi, k, h, bits_w, acts.shape[0], acts.shape[1],
                                    coeffs.shape[1], acts, coeffs, out):
            raise ValueError(self.err())
        return out

    def latticequant_forward(self, G, P, k, h, acts, coeffs, lo=-1.0, hi=1.0):
        acts = np.ascontiguousarray(acts, dtype=np.float64)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        out = np.zeros((acts.shape[0], coeffs.shape[1]))
        if self.lib.ref_latticequant_forward(G, P, lo, hi, k, h, acts.shape[0], acts.shape[1],
                                             coeffs.shape[1], acts, coeffs, out):
            raise ValueError(self.err())
        return out

    def im2col(self, x, kernel, stride, padding):
        x = np.ascontiguousarray(x, dtype=np.float64)
        Cc, H, W = x.shape
        Ho = (H + 2 * padding - kernel) // stride + 1
        Wo = (W + 2 * padding - kernel) // stride + 1
        out = np.zeros((max(Ho, 0) * max(Wo, 0), kernel * kernel * Cc))
        if self.lib.ref_im2col(x, Cc, H, W, kernel, stride, padding, out):
            raise ValueError(self.err())
        return out

    def conv_forward(self, G, P, x, coeffs, c_out, kernel, stride, padding, mode=0, k=8, h=8,
                     bits_w=32, lo=-1.0, hi=1.0):
        x = np.ascontiguousarray(x, dtype=np.float64)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        Cc, H, W = x.shape
        Ho = (H + 2 * padding - kernel) // stride + 1
        Wo = (W + 2 * padding - kernel) // stride + 1
        out = np.zeros((c_out, Ho, Wo))
        if self.lib.ref_conv_forward(G, P, lo, hi, mode, k, h, bits_w, Cc, H, W, c_out, kernel,
                                     stride, padding, x, coeffs, out):
            raise ValueError(self.err())
        return out

    def graph_forward(self, text, coeffs, inputs, n_out, k=8, h=8, bits_w=8, threads=1):
        """Harness composition of reference functions for extended descriptors
        (residual blocks, global average pool, floor-stride convs); LUT mode."""
        inputs = np.ascontiguousarray(inputs, dtype=np.float64)
        cs = [np.ascontiguousarray(c, dtype=np.float64) for c in coeffs]
        ptrs = (C.c_void_p * len(cs))(*[c.ctypes.data for c in cs])
        out = np.zeros((inputs.shape[0], n_out))
        if self.lib.ref_graph_forward(text.encode(), ptrs, k, h, bits_w, inputs.shape[0], inputs,
                                      n_out, out, threads):
            raise ValueError(self.err())
        return out

    def spline_tables(self, G, P, coeffs, n_in, n_out, bits_a, h, kernel=0, stride=1, padding=0,
                      lo=-1.0, hi=1.0):
        """build_spline_tables for a linear (kernel=0; n_in inputs) or conv layer
        (n_in = c_in); returns the same dict as Oracle.spline_tables plus bits."""
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        rows = n_in * (kernel * kernel if kernel else 1)
        vals = np.zeros(rows * n_out << bits_a, dtype=np.uint8)
        qd, qi = np.zeros(2), np.zeros(4, dtype=np.int64)
        bits = self.lib.ref_spline_tables(G, P, lo, hi, n_in, n_out, kernel, stride, padding,
                                          coeffs.ravel(), bits_a, h, vals, vals.size, qd, qi)
        if bits < 0:
            raise ValueError(self.err())
        return {"values": vals.reshape(rows, n_out, 1 << bits_a), "qp_d": qd, "qp_i": qi,
                "bits_a": bits_a, "h": h, "n_in": rows, "n_out": n_out, "stored_bits": bits}

    def spline_forward(self, t, acts):
        acts = np.ascontiguousarray(acts, dtype=np.float64)
        out = np.zeros((acts.shape[0], t["n_out"]))
        if self.lib.ref_spline_table_forward(t["n_in"], t["n_out"], t["bits_a"], t["h"],
                                             np.ascontiguousarray(t["values"]).ravel(), t["qp_d"],
                                             t["qp_i"], acts.shape[0], acts, out):
            raise ValueError(self.err())
        return out

    def st_model_forward(self, text, coeffs, inputs, n_out, bits_a, h, threads=1, chunk=256,
                         reps=1):
        """model_forward in spline-table mode with the tables built once; returns
        (logits, seconds of the `reps` forwards alone)."""
        inputs = np.ascontiguousarray(inputs, dtype=np.float64)
        cs = [np.ascontiguousarray(c, dtype=np.float64) for c in coeffs]
        ptrs = (C.c_void_p * len(cs))(*[c.ctypes.data for c in cs])
        out = np.zeros((inputs.shape[0], n_out))
        sec = C.c_double()
        if self.lib.ref_st_model_forward(text.encode(), ptrs, bits_a, h, inputs.shape[0],
                                         inputs.shape[1], inputs, n_out, out, threads, chunk, reps,
                                         C.byref(sec)):
            raise ValueError(self.err())
        return out, sec.value

    def save_container(self, text, coeffs, path, lut_k=0, lut_h=0, st_bits_a=0, st_h=0):
        """save_container of a descriptor-built model (io.hpp:108-211)."""
        cs = [np.ascontiguousarray(c, dtype=np.float64) for c in coeffs]
        ptrs = (C.c_void_p * len(cs))(*[c.ctypes.data for c in cs])
        if self.lib.ref_save_container(text.encode(), ptrs, lut_k, lut_h, st_bits_a, st_h,
                                       str(path).encode()):
            raise ValueError(self.err())

    def load_container(self, path):
        """load_container: (layer count or -6 io / -7 format / -8 checksum, message)."""
        n = self.lib.ref_load_container(str(path).encode())
        return n, (self.err() if n < 0 else "")

    def calibrate_ranges(self, text, coeffs, inputs, n_kan):
        """calibrate_activation_ranges (eval.hpp:289-341): [n_kan, 2] (lo, hi)."""
        inputs = np.ascontiguousarray(inputs, dtype=np.float64)
        cs = [np.ascontiguousarray(c, dtype=np.float64) for c in coeffs]
        ptrs = (C.c_void_p * len(cs))(*[c.ctypes.data for c in cs])
        out = np.zeros((n_kan, 2))
        if self.lib.ref_calibrate_ranges(text.encode(), ptrs, inputs.shape[0], inputs.shape[1], inputs,
                                         out) < 0:
            raise ValueError(self.err())
        return out

    def fakequant_calibrated_forward(self, text, coeffs, inputs, n_out, bits_w, bits_a, bits_b, ranges):
        inputs = np.ascontiguousarray(inputs, dtype=np.float64)
        cs = [np.ascontiguousarray(c, dtype=np.float64) for c in coeffs]
        ptrs = (C.c_void_p * len(cs))(*[c.ctypes.data for c in cs])
        rg = np.ascontiguousarray(ranges, dtype=np.float64)
        out = np.zeros((inputs.shape[0], n_out))
        if self.lib.ref_fakequant_calibrated_forward(text.encode(), ptrs, bits_w, bits_a, bits_b, rg,
                                                     inputs.shape[0], inputs.shape[1], inputs, n_out, out):
            raise ValueError(self.err())
        return out

    def linear_backward(self, G, P, acts, coeffs, dout, lo=-1.0, hi=1.0):
        """kan_linear_backward (train.hpp:131-136): (dcoeffs, dinputs)."""
        acts = np.ascontiguousarray(acts, dtype=np.float64)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        dout = np.ascontiguousarray(dout, dtype=np.float64)
        dc = np.zeros(coeffs.shape)
        di = np.zeros(acts.shape)
        if self.lib.ref_linear_backward(G, P, lo, hi, acts.shape[0], acts.shape[1], coeffs.shape[1], acts,
                                        coeffs, dout, dc, di):
            raise ValueError(self.err())
        return dc, di

    def train(self, text, coeffs, inputs, labels, lr, momentum, epochs, batch, seed=0):
        """train (train.hpp:247-462): (updated coefficients, last epoch loss)."""
        inputs = np.ascontiguousarray(inputs, dtype=np.float64)
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        cs = [np.ascontiguousarray(c, dtype=np.float64) for c in coeffs]
        outs = [np.zeros_like(c) for c in cs]
        pin = (C.c_void_p * len(cs))(*[c.ctypes.data for c in cs])
        pout = (C.c_void_p * len(outs))(*[o.ctypes.data for o in outs])
        loss = C.c_double()
        if self.lib.ref_train(text.encode(), pin, pout, inputs.shape[0], inputs.shape[1], inputs, labels, lr,
                              momentum, epochs, batch, seed, C.byref(loss)):
            raise ValueError(self.err())
        return outs, loss.value

    def softmax_ce(self, logits, labels):
        logits = np.ascontiguousarray(logits, dtype=np.float64)
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        d = np.zeros(logits.shape)
        loss = C.c_double()
        if self.lib.ref_softmax_ce(logits.shape[0], logits.shape[1], logits, labels, d, C.byref(loss)):
            raise ValueError(self.err())
        return loss.value, d

    def validate_descriptor(self, text: str) -> int:
        n = self.lib.ref_validate_descriptor(text.encode())
        if n < 0:
            raise ValueError(self.err())
        return n

    def model_forward(self, text, coeffs, inputs, n_out, mode=0, k=8, h=8, bits_w=8,
                      threads=1, chunk=256):
        inputs = np.ascontiguousarray(inputs, dtype=np.float64)
        cs = [np.ascontiguousarray(c, dtype=np.float64) for c in coeffs]
        ptrs = (C.c_void_p * len(cs))(*[c.ctypes.data for c in cs])
        out = np.zeros((inputs.shape[0], n_out))
        if self.lib.ref_model_forward(text.encode(), ptrs, mode, k, h, bits_w, inputs.shape[0],
                                      inputs.shape[1], inputs, n_out, out, threads, chunk):
            raise ValueError(self.err())
        return out

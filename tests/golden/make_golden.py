"""Generate the committed golden vectors from the REFERENCE ITSELF.

Run in the build container (where /root/reference exists and
oracle/_ref/libkantize_ref.so was compiled from it by oracle/Makefile):

    python tests/golden/make_golden.py

Every array below is produced by a reference function (via oracle/ref_shim.cpp);
nothing comes from the restatement under test.  Output: tests/golden/reference_golden.npz
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Ref  # noqa: E402


def main():
    r = Ref()
    out = {}
    # build_bspline_lut entries (lut.hpp:103-131) for every P, k, h the configs touch
    for P in (1, 2, 3):
        for k in (1, 2, 3, 4, 8):
            for h in (2, 3, 4, 8):
                e, mb = r.lut(P, k, h)
                out[f"lut_P{P}_k{k}_h{h}"] = e
                out[f"lutbits_P{P}_k{k}_h{h}"] = np.array([mb])
    # lattice levels of an edge-case fp32 vector (clamp + ActivationLattice::quantize)
    rng = np.random.default_rng(20260317)
    x = np.concatenate([
        rng.uniform(-1.3, 1.3, 4000),
        np.linspace(-1.0, 1.0, 1281),
        [0.0, -0.0, 1.0, -1.0, np.nextafter(1.0, 0), np.nextafter(-1.0, 0), 1e30, -1e30,
         np.inf, -np.inf, np.nan, 1e-40],
    ]).astype(np.float32)
    out["levels_x"] = x
    for (G, k) in ((5, 8), (10, 8), (5, 4), (5, 3), (5, 2), (3, 4)):
        out[f"levels_G{G}_k{k}"] = r.levels(G, 3, k, x)
    # lut_basis_lookup for every level of (G=5, P=3, k=8, h=8) and (G=10, k=8, h=8)
    for (G, k, h) in ((5, 8, 8), (10, 8, 8), (5, 8, 3), (5, 4, 4)):
        L = G << k
        vals = np.zeros((L + 1, 4), dtype=np.uint8)
        start = np.zeros(L + 1, dtype=np.int32)
        cnt = np.zeros(L + 1, dtype=np.int32)
        for a in range(L + 1):
            v, s = r.lut_lookup(G, 3, k, h, a)
            vals[a, :len(v)] = v
            start[a], cnt[a] = s, len(v)
        out[f"lookup_G{G}_k{k}_h{h}_vals"] = vals
        out[f"lookup_G{G}_k{k}_h{h}_start"] = start
        out[f"lookup_G{G}_k{k}_h{h}_count"] = cnt
    # layer forwards: kan_linear_forward (fp64) and tabulated_kan_forward (k8,h8,w8)
    acts = rng.uniform(-1.1, 1.1, (16, 24))
    coeffs = rng.normal(0, 0.1, (24 * 8, 6))
    out["fwd_acts"] = acts
    out["fwd_coeffs"] = coeffs
    out["fwd_linear_G5"] = r.linear_forward(5, 3, acts, coeffs)
    out["fwd_lut_G5_k8_h8_w8"] = r.lut_forward(5, 3, 8, 8, 8, acts, coeffs)
    out["fwd_lut_G5_k4_h4_w4"] = r.lut_forward(5, 3, 4, 4, 4, acts, coeffs)
    # basis known answer: cox_de_boor(0.0) on (G=3, P=3) = (0, 1/48, 23/48, 23/48, 1/48, 0)
    b, s = r.cox_de_boor(3, 3, 0.0)
    out["basis_G3_at0"] = b
    # quant params (-1, 1, 8) -> s = 2/255, z = 128 (test_quant.cpp:12-19)
    out["qp_m1_1_8"] = np.array(r.quant_params(-1.0, 1.0, 8))
    # im2col of a 2x3x3 input, k=3 s=1 p=1 (layers.hpp:126-154)
    img = rng.uniform(-1, 1, (2, 3, 3))
    out["im2col_in"] = img
    out["im2col_k3s1p1"] = r.im2col(img, 3, 1, 1)
    np.savez_compressed(os.path.join(os.path.dirname(__file__), "reference_golden.npz"), **out)
    print(f"wrote {len(out)} arrays")


if __name__ == "__main__":
    main()

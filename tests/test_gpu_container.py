"""GPU: an engine loaded from a .kant container (kan_engine_load) runs exactly
what an engine built from the same descriptor + coefficients runs, and the
reference's own container (oracle/_ref save_container) drives it: LUT path
with the stored LUT, spline-table path with the stored tables (bit-exact vs
the oracle)."""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2603_17230_b200 import Engine, EvalOptions, W_PER_TENSOR_ASYM, load_container, save_container  # noqa: E402

DESC = {"name": "m", "grid": {"intervals": 5, "degree": 3}, "input": [40],
        "layers": [{"type": "linear", "n_in": 40, "n_out": 24}, {"type": "linear", "n_in": 24, "n_out": 10}]}


def _ws(seed=3):
    rng = np.random.default_rng(seed)
    return [rng.normal(0, 0.1, (40 * 8, 24)), rng.normal(0, 0.1, (24 * 8, 10))]


def test_loaded_engine_matches_built_engine(tmp_path):
    ws = _ws()
    p = tmp_path / "m.kant"
    save_container(p, DESC, ws)
    x = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, (300, 40)).astype(np.float32)).cuda()
    opts = EvalOptions(mode="bspline-lut", lut_k=8, lut_h=8, bits_w=8, w_scheme=W_PER_TENSOR_ASYM)
    a = Engine.load(p)
    a.configure(opts)
    b = Engine(DESC)
    for i, w in enumerate(ws):
        b.set_coeffs(i, w.astype(np.float32).astype(np.float64))
    b.configure(opts)
    np.testing.assert_array_equal(a.model_forward(x).cpu().numpy(), b.model_forward(x).cpu().numpy())


def test_reference_container_with_tables_drives_both_table_paths(ref, oracle, tmp_path):
    ws = _ws(5)
    p = tmp_path / "r.kant"
    ref.save_container(json.dumps(DESC), ws, p, lut_k=4, lut_h=6, st_bits_a=6, st_h=7)
    e = Engine.load(p)
    x = np.random.default_rng(1).uniform(-1.1, 1.1, (200, 40)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    # spline-table mode on the stored tables
    e.configure(EvalOptions(mode="spline-table", lut_k=6, lut_h=7))
    y = e.model_forward(xd).cpu().numpy()
    ws32 = [w.astype(np.float32).astype(np.float64) for w in ws]
    tabs = oracle.spline_model_tables(DESC, ws, 6, 7)  # the reference tabulated its fp64 coefficients
    want = oracle.spline_model_forward(DESC, tabs, x.astype(np.float64)).astype(np.float32)
    np.testing.assert_array_equal(y, want)
    # LUT mode with the stored (k=4, h=6) table: the reference's model_forward
    e.configure(EvalOptions(mode="bspline-lut", lut_k=4, lut_h=6, bits_w=8, w_scheme=W_PER_TENSOR_ASYM))
    np.testing.assert_array_equal(e.lut(), load_container(p)["lut"]["entries"])
    y = e.model_forward(xd).cpu().numpy().astype(np.float64)
    r = ref.model_forward(json.dumps(DESC), ws32, x.astype(np.float64), 10, mode=2, k=4, h=6, bits_w=8)
    assert np.abs(y - r).max() <= 1e-6 * max(1.0, np.abs(r).max())

"""The .kant container (io.hpp:99-350) on the host: the engine's reader and
writer against the reference's own save_container / load_container (oracle/_ref)
and the reference's known answers (test_io.cpp)."""
import json
import os

import numpy as np
import pytest

from paper_2603_17230_b200 import crc32, load_container, save_container
from paper_2603_17230_b200.engine import KanError

MLP = {"name": "m", "grid": {"intervals": 3, "degree": 3}, "input": [12],
       "layers": [{"type": "linear", "n_in": 12, "n_out": 5}, {"type": "linear", "n_in": 5, "n_out": 3}]}
LEKAN = {"name": "LeKAN", "grid": {"intervals": 3, "degree": 3}, "input": [1, 28, 28],
         "layers": [{"type": "conv", "c_in": 1, "c_out": 6, "kernel": 5, "stride": 1, "padding": 0},
                    {"type": "maxpool", "window": 2},
                    {"type": "conv", "c_in": 6, "c_out": 16, "kernel": 5, "stride": 1, "padding": 0},
                    {"type": "maxpool", "window": 2}, {"type": "flatten"},
                    {"type": "linear", "n_in": 256, "n_out": 10}]}


def _coeffs(desc, seed):
    rng = np.random.default_rng(seed)
    nb = desc["grid"]["intervals"] + desc["grid"]["degree"]
    out = []
    for l in desc["layers"]:
        if l["type"] == "linear":
            out.append(rng.uniform(-1, 1, (l["n_in"] * nb, l["n_out"])))
        elif l["type"] == "conv":
            out.append(rng.uniform(-1, 1, (l["c_in"] * l["kernel"] ** 2 * nb, l["c_out"])))
    return out


def test_crc32_reference_value():
    assert crc32(b"123456789") == 0xCBF43926  # test_io.cpp:35-38


def test_frozen_byte_layout(tmp_path):
    """test_io.cpp:145-165: a fixed tiny model serializes to exactly 275 bytes
    with CRC 0xB9242D23."""
    desc = {"name": "g", "grid": {"intervals": 2, "degree": 1}, "input": [2],
            "layers": [{"type": "linear", "n_in": 2, "n_out": 2}]}
    w = (0.125 * (np.arange(3 * 2 * 2) - 3.0)).reshape(6, 2)
    p = tmp_path / "golden.kant"
    save_container(p, desc, [w])
    b = p.read_bytes()
    assert len(b) == 275
    assert crc32(b) == 0xB9242D23


@pytest.mark.parametrize("desc,lut,st", [(MLP, None, None), (MLP, (4, 8), (4, 6)), (LEKAN, (8, 3), None),
                                         (LEKAN, None, (5, 7))])
def test_engine_writer_matches_reference_bytes_and_reader_round_trips(ref, oracle, tmp_path, desc, lut, st):
    ws = _coeffs(desc, 77)
    text = json.dumps(desc)
    pr, pe = tmp_path / "ref.kant", tmp_path / "eng.kant"
    ref.save_container(text, ws, pr, lut_k=lut[0] if lut else 0, lut_h=lut[1] if lut else 0,
                       st_bits_a=st[0] if st else 0, st_h=st[1] if st else 0)
    c = load_container(pr)
    assert c["descriptor"]["input"] == desc["input"]
    assert [l["type"] for l in c["descriptor"]["layers"]] == [l["type"] for l in desc["layers"]]
    for a, b in zip(c["coeffs"], ws):
        np.testing.assert_array_equal(a, b.astype(np.float32).astype(np.float64).ravel())
    if lut:
        assert c["lut"]["k"] == lut[0] and c["lut"]["h"] == lut[1]
        np.testing.assert_array_equal(c["lut"]["entries"], oracle.lut(desc["grid"]["degree"], *lut))
    else:
        assert c["lut"] is None
    if st:
        g = oracle.grid(desc["grid"]["intervals"], desc["grid"]["degree"])
        assert len(c["spline_tables"]) == len(ws)
        for t, w in zip(c["spline_tables"], ws):
            n_out = w.shape[1]
            want = oracle.spline_tables(g, w, w.shape[0] // (desc["grid"]["intervals"] + 3), n_out, *st)
            np.testing.assert_array_equal(t["values"], want["values"].ravel())
            np.testing.assert_array_equal(t["qp_d"], want["qp_d"])
            np.testing.assert_array_equal(t["qp_i"], want["qp_i"])
    # the engine writes the same bytes from what it read
    save_container(pe, c["descriptor"], c["coeffs"],
                   lut=c["lut"], spline_tables=c["spline_tables"] or None)
    assert pe.read_bytes() == pr.read_bytes()
    assert ref.load_container(pe)[0] == len(desc["layers"])


def test_damaged_files(tmp_path):
    """test_io.cpp:73-115: missing -> io_error, truncated / bad magic / unknown
    version (named) -> format_error, payload corruption -> checksum_error."""
    p = tmp_path / "d.kant"
    save_container(p, MLP, _coeffs(MLP, 5))
    good = p.read_bytes()
    with pytest.raises(OSError):
        load_container(str(p) + ".nope")
    p.write_bytes(good[:len(good) // 2])
    with pytest.raises(ValueError) as ei:
        load_container(p)
    assert ei.value.args[0].status == 7
    p.write_bytes(b"X" + good[1:])
    with pytest.raises(ValueError) as ei:
        load_container(p)
    assert ei.value.args[0].status == 7
    p.write_bytes(good[:4] + bytes([9]) + good[5:])
    with pytest.raises(ValueError) as ei:
        load_container(p)
    assert ei.value.args[0].status == 7 and "9" in str(ei.value)
    bad = bytearray(good)
    bad[-20] ^= 0x40
    p.write_bytes(bytes(bad))
    with pytest.raises(ValueError) as ei:
        load_container(p)
    assert ei.value.args[0].status == 8


def test_extension_descriptors_have_no_container_form(tmp_path):
    from paper_2603_17230_b200 import configs
    wl = configs.get("c5")
    with pytest.raises(NotImplementedError):
        save_container(tmp_path / "x.kant", wl.descriptor(), [np.zeros(1)] * wl.n_kan)

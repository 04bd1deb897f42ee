"""Sweep host logic (sweep.hpp) against the reference's known answers
(test_sweep.cpp:28-80, test_cost.cpp:151-152); no GPU."""
import pytest

from paper_2603_17230_b200.sweep import (SweepSpec, csv_header, enumerate_configs, fp32_coeff_bits,
                                         lut_memory_bits, pareto_front, spline_table_bits)


def test_configuration_enumeration():
    assert len(enumerate_configs(SweepSpec([8], [8], [2, 3, 4]))) == 3
    full = [2, 3, 4, 5, 6, 7, 8, 32]
    assert len(enumerate_configs(SweepSpec(full, full, full))) == 512
    a = enumerate_configs(SweepSpec([8, 2], [4, 3], [2, 8]))
    assert [(c.bits_w, c.bits_a, c.bits_b) for c in a] == [
        (8, 4, 2), (8, 4, 8), (8, 3, 2), (8, 3, 8), (2, 4, 2), (2, 4, 8), (2, 3, 2), (2, 3, 8)]
    assert len(enumerate_configs(SweepSpec([8], [4, 32], [3, 32], ["bspline-lut"]))) == 1
    st = enumerate_configs(SweepSpec([2, 4, 8], [4], [6], ["spline-table"]))
    assert len(st) == 1 and st[0].bits_w == 32
    with pytest.raises(ValueError):
        enumerate_configs(SweepSpec([], [8], [8]))
    with pytest.raises(ValueError):
        enumerate_configs(SweepSpec(modes=["telepathy"]))


def test_costs_and_pareto():
    mlp1 = {"grid": {"intervals": 3, "degree": 3}, "input": [784],
            "layers": [{"type": "linear", "n_in": 784, "n_out": 10}]}
    assert spline_table_bits(mlp1, 4, 6) == 752640  # test_cost.cpp:151
    assert spline_table_bits(mlp1, 8, 8) == 16056320  # test_cost.cpp:152
    assert fp32_coeff_bits(mlp1) == 784 * 10 * 6 * 32
    assert lut_memory_bits(3, 8, 8) == 256 * 2 * 8
    assert pareto_front([0.9, 0.8, 0.9, 0.5], [10, 5, 20, 1]) == [0, 1, 3]
    assert csv_header().startswith("model,mode,bw_w,bw_a,bw_b,accuracy")

"""The measurement model of bench.py (CPU): the SURVEY 8(d) byte model per
level, the per-direction roofline split and the harmonic mean."""

import os
import sys
from dataclasses import dataclass

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


@dataclass
class Rec:
    n_f: int
    scanned_edges: int
    direction: str
    executed_direction: str
    wall_time: float


def test_level_bytes_follow_the_byte_model():
    n_dev, n_plus = 1 << 20, 900_000
    levels = [Rec(1, 10, "top_down", "top_down", 1e-6),
              Rec(9, 5000, "bottom_up", "bottom_up", 2e-6),
              Rec(700, 40, "bottom_up", "top_down", 3e-6)]
    lb = bench.level_bytes(levels, n_dev, n_plus)
    # TD: |F|*20 + 4*E + 8*n_next
    assert lb[0] == ("top_down", 1 * 20 + 4 * 10 + 8 * 9, 1e-6)
    # BU: 3*n_dev/8 + 8*U + 4*C + 4*n_next, U = n_plus - reached (frontier included)
    assert lb[1] == ("bottom_up", 3 * (n_dev // 8) + 8 * (n_plus - 10) + 4 * 5000 + 4 * 700, 2e-6)
    # the executed direction decides the model
    assert lb[2][0] == "top_down" and lb[2][1] == 700 * 20 + 4 * 40
    assert bench.algorithmic_bytes(levels, n_dev, n_plus) == sum(b for _, b, _ in lb)


def test_by_direction_split_and_hmean():
    per_root = [[("top_down", 1000, 1e-6), ("bottom_up", 9000, 2e-6)],
                [("top_down", 3000, 1e-6), ("bottom_up", 1000, 1e-6)]]
    d = bench.by_direction(per_root, peak=1.0)
    assert d["top_down"]["levels"] == 2 and d["bottom_up"]["levels"] == 2
    assert np.isclose(d["top_down"]["achieved"], 4000 / 2e-6 / 1e9)
    assert np.isclose(d["bottom_up"]["achieved"], 10000 / 3e-6 / 1e9)
    assert np.isclose(d["bottom_up"]["largest_level"]["bytes_mean"], (9000 + 1000) / 2)
    assert np.isclose(bench.hmean([1.0, 4.0]), 1.6)

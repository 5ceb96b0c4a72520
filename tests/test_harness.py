"""Experiment harness (paper_1808_06357_b200/harness.py), CPU part: the
summary statistics and the output formats, with a stub solver."""
import csv
import json
import os

import numpy as np

import paper_1808_06357_b200 as L
from paper_1808_06357_b200 import harness


class _Stub:
    def __init__(self):
        self.lat = L.Lattice.rank1([1, 34], 55)
        self.dt = 0.01

    def propagate(self, m, record_every, member=0):
        k = np.arange(0, m + 1, record_every)
        return np.stack([k, k * self.dt, 1.0 + 1e-13 * np.sin(k), 2.0 + 1e-9 * np.cos(k)], axis=1)


def test_variation_is_paper_delta():
    assert abs(harness.variation([1.0, 1.0 + 2e-12, 1.0 - 2e-12]) - 4e-12) < 1e-15
    assert harness.variation([]) == 0.0


def test_fit_slope_second_order_and_exact_flag():
    dts = [1 / 8, 1 / 16, 1 / 32, 1 / 64]
    slope, how = harness.fit_slope(dts, [3.0 * d ** 2 for d in dts])
    assert how == "fit" and abs(slope - 2.0) < 1e-12
    assert harness.fit_slope(dts, [1e-16] * 4) == (None, "exact")  # round-off floor excluded


def test_conservation_outputs(tmp_path):
    s = harness.run_conservation(_Stub(), 40, 4, config={"d": 2}, out_dir=str(tmp_path))
    assert s["records"] == 11 and s["lattice_hash"] == f"0x{L.Lattice.rank1([1, 34], 55).hash():016x}"
    assert s["delta_norm"] < 3e-13 and s["delta_energy"] < 1.1e-9
    rows = list(csv.reader(open(os.path.join(tmp_path, "conservation.csv"))))
    assert rows[0] == ["step", "time", "norm", "energy", "dnorm", "denergy"] and len(rows) == 12
    js = json.load(open(os.path.join(tmp_path, "conservation.json")))
    assert js["config"] == {"d": 2} and "sm_100a" in js["tool"]


def test_conservation_m0_is_empty():
    s = harness.run_conservation(_Stub(), 0, 1)
    assert s["records"] == 0 and s["delta_norm"] == 0.0 and s["delta_energy"] == 0.0

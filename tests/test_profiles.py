"""The committed ncu evidence agrees with the bench's algorithmic byte model.

profiles/r1g holds, per streamed config (C2-C4), the bench line and the ncu
DRAM counters of consecutive pass launches inside the step loop. The DESIGN.md
§4 claim is that each pass moves no more than its algorithmic bytes
(`roofline.bytes_per_launch`, `solver.bytes_per_step`); this pins it.
"""
import json
import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(ROOT, "paper_1808_06357_b200", "tools"))
import ncu_traffic  # noqa: E402

PROF = os.path.join(ROOT, "profiles", "r1g")


@pytest.mark.parametrize("cfg", ["C2", "C3", "C4"])
def test_pass_traffic_within_algorithmic_bytes(cfg):
    line = json.loads(open(os.path.join(PROF, f"{cfg}_plain.json")).read().strip().splitlines()[-1])
    r, s = line["roofline"], line["solver"]
    col_alg = r["bytes_per_launch"] if r["kernel"].startswith("col") else s["bytes_per_step"] - r["bytes_per_launch"]
    row_alg = s["bytes_per_step"] - col_alg
    table = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    for side, alg in (("col", col_alg), ("row", row_alg)):
        got = table[f"{cfg}_circulant_{side}"]
        assert 0.75 * alg <= got <= 1.02 * alg, (cfg, side, got, alg)


def test_parser_reads_committed_csv():
    launches = ncu_traffic.load(os.path.join(PROF, "C4_traffic.csv"))
    assert len(launches) == 8
    assert all("dram__bytes_read.sum" in v and "gpu__time_duration.sum" in v for _, v in launches)

"""Fold ncu DRAM captures of configs 2-4 into profiles/ncu_traffic.json.

Reads gpurun_out/<tag>/{C2,C3,C4}_traffic.csv (ncu_traffic.sh) and the
matching *_plain.json bench lines. Step kernels are the fft_pass_kernel
instances whose fifth template argument (program) is 0; the COL pass is the
one whose first argument is 1 and length is the solver's M1, every other step
kernel belongs to the row side. Per-launch traffic is dram read + write; the
row side of a three-level geometry (config 4) is several launches, so its
entry is the mean per row-side launch times (launches_per_step - 1), matching
how bench.py's pass_ms["row"] covers the whole row side.

    python paper_1808_06357_b200/tools/ncu_traffic.py r1g
"""
import csv
import json
import os
import re
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def load(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(text[start:].splitlines()))
    per = defaultdict(dict)
    for r in rows:
        scale = UNIT.get(r.get("Metric Unit", "byte"), 1.0)
        try:
            val = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        per[(int(r["ID"]), r["Kernel Name"])][r["Metric Name"]] = val * (scale if "bytes" in r["Metric Name"] else 1.0)
    return [(k[1], v) for k, v in sorted(per.items())]


def main(tag):
    out_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    table = json.load(open(out_path)) if os.path.exists(out_path) else {}
    for cfg in ("C2", "C3", "C4"):
        base = os.path.join(ROOT, "gpurun_out", tag)
        csvp, jp = os.path.join(base, f"{cfg}_traffic.csv"), os.path.join(base, f"{cfg}_plain.json")
        if not (os.path.exists(csvp) and os.path.exists(jp)):
            print(f"{cfg}: missing capture")
            continue
        line = json.loads(open(jp).read().strip().splitlines()[-1])
        m1, lps = line["solver"]["M1"], line["solver"]["launches_per_step"]
        col, row = [], []
        for name, v in load(csvp):
            t = re.search(r"fft_pass_kernel<([^>]*)>", name)
            if not t:
                continue
            args = [a.strip() for a in t.group(1).split(",")]
            if args[4] != "0":
                continue
            b = v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
            (col if args[0] == "1" and int(args[1]) == m1 else row).append(b)
        if col:
            table[f"{cfg}_circulant_col"] = sum(col) / len(col)
        if row:
            table[f"{cfg}_circulant_row"] = sum(row) / len(row) * max(1, lps - 1)
        print(cfg, "col", col, "row", row)
    json.dump(table, open(out_path, "w"), indent=1)
    print(json.dumps(table, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])

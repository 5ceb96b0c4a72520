"""Fold ncu DRAM captures of configs 2-4 into profiles/ncu_traffic.json.

Reads gpurun_out/<tag>/{C2,C3,C4}_traffic.csv (ncu_traffic.sh) and the
matching *_plain.json bench lines. The step COL pass is the
fft_pass4_kernel / fft_pass_kernel instance whose first template argument is
1 (COL), length the solver's M1 and (v1) program, the fifth argument, 0; the row side of that step is the
launches_per_step - 1 launches right before it (one ROW pass, or at config 4's
three-level geometry COL-Ma, ROW-Mb, COL-Ma), matching how bench.py's
pass_ms["row"] covers the whole row side. Traffic is dram read + write.

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


def main(tag, configs=("C2", "C3", "C4")):
    """Entries carry the geometry and kernel family they were captured on
    (bench.py emits roofline.traffic only when they match the run) and the
    source file; a capture with no step COL launch or fewer than 2 samples
    per side fails instead of silently keeping old values."""
    out_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    table = json.load(open(out_path)) if os.path.exists(out_path) else {}
    table = {k: v for k, v in table.items() if isinstance(v, dict)}  # drop pre-r2 bare numbers
    bad = []
    for cfg in configs:
        base = os.path.join(ROOT, "gpurun_out", tag)
        csvp, jp = os.path.join(base, f"{cfg}_traffic.csv"), os.path.join(base, f"{cfg}_plain.json")
        if not (os.path.exists(csvp) and os.path.exists(jp)):
            print(f"{cfg}: missing capture")
            bad.append(cfg)
            continue
        line = json.loads(open(jp).read().strip().splitlines()[-1])
        sol = line["solver"]
        m1, lps = sol["M1"], sol["launches_per_step"]
        launches = []
        for name, v in load(csvp):
            if "fft_pass4s_kernel" in name:  # lean single-transform pass (three-level inner passes): row side
                launches.append((False, v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)))
                continue
            t = re.search(r"fft_pass(4?)_kernel<([^>]*)>", name)
            if t:
                # v1: <axis, L, B, NT, prog, sign, minb>; pass4 (always the double program):
                # <axis, L, B, LPT, PP, NT, sign, TW, DK, minb>
                args = [re.sub(r"\((int|bool)\)", "", a).strip() for a in t.group(2).split(",")]
                b = v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
                step_col = args[0] == "1" and int(args[1]) == m1 and (t.group(1) == "4" or args[4] == "0")
                launches.append((step_col, b))
        cols = [i for i, (is_col, _) in enumerate(launches) if is_col]
        col = [launches[i][1] for i in cols]
        # the row side of one step = the lps-1 launches right before a step COL launch
        row = [sum(b for _, b in launches[i - (lps - 1):i]) for i in cols if i >= lps - 1]
        print(cfg, "col", col, "row", row)
        if len(col) < 2 or len(row) < 2:
            bad.append(cfg)
            continue
        meta = {"M1": sol["M1"], "M2": sol["M2"], "group": sol["group"], "kernel": sol.get("pass_kernel"),
                "source": f"profiles/{tag}/{cfg}_traffic.csv"}
        table[f"{cfg}_circulant_col"] = {"bytes": sum(col) / len(col), "samples": len(col), **meta}
        table[f"{cfg}_circulant_row"] = {"bytes": sum(row) / len(row), "samples": len(row), **meta}
    json.dump(table, open(out_path, "w"), indent=1)
    print(json.dumps(table, indent=1))
    if bad:
        sys.exit(f"ncu_traffic: no usable step-pass capture for {bad}")


if __name__ == "__main__":
    main(sys.argv[1], tuple(sys.argv[2:]) or ("C2", "C3", "C4"))

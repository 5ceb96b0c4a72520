"""Turn a round's raw GPU artefacts (gpurun_out/<tag>/) into the committed
profile summaries (profiles/<tag>/): launch-list shares, ncu --set full key
metrics of the hot pass kernels, steady-state (no cache flush) DRAM bytes,
and profiles/ncu_traffic.json (per-launch DRAM bytes bench.py reports as
roofline.traffic).

    python paper_1808_06357_b200/tools/summarize_profiles.py r1 [--config C1 --method circulant]
"""
import argparse
import csv
import io
import json
import os
import shutil
import subprocess
from collections import defaultdict

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))


def launch_list(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')]
    if not start:
        return []
    rows = list(csv.reader(lines[start[0]:]))
    hdr = rows[0]
    I = {h: i for i, h in enumerate(hdr)}
    out = []
    for r in rows[1:]:
        if r[I["Metric Name"]] == "gpu__time_duration.sum":
            v = float(r[I["Metric Value"]])
            unit = r[I["Metric Unit"]]
            ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
            out.append((r[I["Kernel Name"]], ns))
    return out


def short(name):
    name = name.replace("lattdse_dev::", "").replace("(PassArgs)", "").replace("(lattdse_dev::PassArgs)", "")
    return name[:80]


def ncu_raw(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    return rows[0], rows[1], rows[2:]


KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_pct"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex_pct"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
]


def to_bytes(v, unit):
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--config", default="C1")
    ap.add_argument("--method", default="circulant")
    args = ap.parse_args()
    src = os.path.join(ROOT, "gpurun_out", args.tag)
    dst = os.path.join(ROOT, "profiles", args.tag)
    os.makedirs(dst, exist_ok=True)
    md = [f"# Profiles {args.tag} -- {args.config} ({args.method})", ""]

    # 1. launch list
    ll = launch_list(os.path.join(src, "launches.csv"))
    if ll:
        shutil.copy(os.path.join(src, "launches.csv"), os.path.join(dst, "launches.csv"))
        agg = defaultdict(lambda: [0, 0.0])
        for n, ns in ll:
            agg[short(n)][0] += 1
            agg[short(n)][1] += ns
        tot = sum(v[1] for v in agg.values())
        md += ["## Launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)", "",
               "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for n, (c, ns) in sorted(agg.items(), key=lambda x: -x[1][1]):
            md.append(f"| `{n}` | {c} | {ns / 1e3:.1f} | {100 * ns / tot:.1f}% |")
        md.append("")

    # 2. full capture
    traffic = {}
    rep = os.path.join(src, f"prof_{args.config.lower()}.ncu-rep")
    if os.path.exists(rep):
        hdr, units, rows = ncu_raw(rep)
        md += ["## ncu --set full (cold cache: ncu flushes caches between replays)", ""]
        for r in rows:
            name = short(r[hdr.index("Kernel Name")])
            md.append(f"### `{name}`")
            for k, lab in KEYS:
                if k in hdr:
                    md.append(f"- {lab}: {r[hdr.index(k)]} {units[hdr.index(k)]}")
            stalls = []
            for i, h in enumerate(hdr):
                if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                    try:
                        stalls.append((float(r[i]), h[34:-23]))
                    except ValueError:
                        pass
            md.append("- stalls per issued instruction: " +
                      ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)[:6]))
            md.append("")
            axis = "col" if "<1," in name or "<(int)1," in name else "row"
            rd = to_bytes(r[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")])
            wr = to_bytes(r[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
            traffic[f"{args.config}_{args.method}_{axis}"] = rd + wr

    # 3. steady state
    st = os.path.join(src, "ncu_steady.csv")
    if os.path.exists(st):
        lines = open(st).read().splitlines()
        start = [i for i, l in enumerate(lines) if l.startswith('"ID"')]
        if start:
            rows = list(csv.reader(lines[start[0]:]))
            I = {h: i for i, h in enumerate(rows[0])}
            md += ["## Steady state inside the step loop (ncu --cache-control none)", "",
                   "| launch | kernel | metric | value |", "|---|---|---|---|"]
            for r in rows[1:]:
                md.append(f"| {r[I['ID']]} | `{short(r[I['Kernel Name']])}` | {r[I['Metric Name']]} | "
                          f"{r[I['Metric Value']]} {r[I['Metric Unit']]} |")
            md.append("")
    open(os.path.join(dst, "README.md"), "w").write("\n".join(md) + "\n")
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    cur = json.load(open(tp)) if os.path.exists(tp) else {}
    cur.update(traffic)
    json.dump(cur, open(tp, "w"), indent=1)
    print("wrote", dst, traffic)


if __name__ == "__main__":
    main()

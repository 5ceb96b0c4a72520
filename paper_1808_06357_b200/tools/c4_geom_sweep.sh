#!/usr/bin/env bash
# Config-4 geometry sweep on one GPU (LATTDSE_GEOM = M1 x Ma x Mb), 8 Strang
# steps per bench step; prints us/step and the COL / row-side pass times.
cd "$(dirname "$0")/../.."
for g in "$@"; do
  LATTDSE_GEOM=$g timeout 600 python bench.py --config C4 --steps 1 --warmup 1 --m 8 --no-cpu > gpurun_out/c4g_$g.log 2>&1
  python - "$g" <<'PY'
import json, sys
g = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/c4g_{g}.log").read().strip().splitlines()[-1])
    s = d["solver"]
    print(f"{g:18s} M={s['M']} {d['us_per_strang_step']/1e3:.1f} ms/step col={d['roofline']['pass_ms']['col']:.1f} row-side={d['roofline']['pass_ms']['row']:.1f} ms")
except Exception as e:
    print(g, "FAILED", open(f"gpurun_out/c4g_{g}.log").read()[-400:])
PY
done

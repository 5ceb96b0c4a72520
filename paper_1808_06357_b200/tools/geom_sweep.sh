#!/usr/bin/env bash
# Geometry sweep for any config on one GPU (LATTDSE_GEOM = M1xM2 or M1xMaxMb):
#   geom_sweep.sh C3 64 486x1080 405x1296 ...
# (m Strang steps per bench step); prints us/step and the COL / ROW pass times.
cd "$(dirname "$0")/../.."
cfg=$1; m=$2; shift 2
for g in "$@"; do
  LATTDSE_GEOM=$g timeout 600 python bench.py --config "$cfg" --steps 2 --warmup 3 --m "$m" --no-cpu > "gpurun_out/g_${cfg}_$g.log" 2>&1
  python - "$cfg" "$g" <<'PY'
import json, sys
cfg, g = sys.argv[1], sys.argv[2]
f = f"gpurun_out/g_{cfg}_{g}.log"
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    s = d["solver"]
    print(f"{cfg} {g:18s} M={s['M']} {d['us_per_strang_step']:.1f} us/step col={d['roofline']['pass_ms']['col']*1e3:.1f} row={d['roofline']['pass_ms']['row']*1e3:.1f} us  value={d['value']:.4e}")
except Exception as e:
    print(cfg, g, "FAILED", open(f).read()[-400:])
PY
done

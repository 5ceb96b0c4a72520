#!/usr/bin/env bash
# Config 3 ensemble group-size sweep (LATTDSE_GROUP) at two geometries.
cd "$(dirname "$0")/../.."
for g in ${GEOMS:-486x1080 1080x486}; do
  for grp in ${GRPS:-0 4 6 12 16 24 32}; do
    LATTDSE_GEOM=$g LATTDSE_GROUP=$grp timeout 600 python bench.py --config C3 --steps 2 --warmup 3 --m 64 --no-cpu > "gpurun_out/c3g_${g}_$grp.log" 2>&1
    python -c "
import json
d = json.loads(open('gpurun_out/c3g_${g}_$grp.log').read().strip().splitlines()[-1])
print('$g group=$grp(auto=0)', d['solver']['group'], round(d['us_per_strang_step'], 1), 'us/step', '%.4e' % d['value'])" || tail -3 "gpurun_out/c3g_${g}_$grp.log"
  done
done

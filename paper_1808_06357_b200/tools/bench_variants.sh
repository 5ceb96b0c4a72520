#!/usr/bin/env bash
# Quick A/B of pass-kernel variants on the bench workload (GPU box).
# usage: tools/bench_variants.sh "TAG:ENV=.. ENV=.." ...   (extra bench args via $EXTRA)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for spec in "$@"; do
  tag=${spec%%:*}; envs=${spec#*:}
  env $envs timeout 200 python bench.py --steps 3 --warmup 3 --no-cpu $EXTRA > gpurun_out/bench_$tag.log 2>&1
  python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/bench_{tag}.log").read().strip().splitlines()[-1])
    print(f"{tag:10s} {d['value']:.3e} pt-steps/s  {d['us_per_strang_step']:.1f} us/step  col={d['roofline']['pass_ms']['col']*1e3:.1f}us row={d['roofline']['pass_ms']['row']*1e3:.1f}us  M={d['solver']['M']} {d['solver']['M1']}x{d['solver']['M2']}")
except Exception as e:
    print(tag, "FAILED", open(f"gpurun_out/bench_{tag}.log").read()[-600:])
PY
done

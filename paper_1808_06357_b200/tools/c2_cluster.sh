#!/usr/bin/env bash
# Config 2 with the opt-in cluster COL pass: parity tests, then the bench per
# cluster size (0 = plain pass).
set -u
cd "$(dirname "$0")/../.."
T=gpurun_out/$1
mkdir -p "$T"
timeout 900 python -m pytest tests -m gpu -q -x -k "cluster or config2" > "$T/pytest_cluster.log" 2>&1; echo "pytest rc=$?" >> "$T/status_c2.txt"
for v in 0 2 4 8; do
  LATTDSE_CLUSTER_COL=$v timeout 600 python bench.py --config C2 --steps 2 --warmup 3 --m 64 --no-cpu > "$T/c2c_$v.json" 2> "$T/c2c_$v.err"; echo "c2 $v rc=$?" >> "$T/status_c2.txt"
done
cat "$T/status_c2.txt"

#!/usr/bin/env bash
# DRAM traffic per pass launch for configs 2-4 (GPU box, one call), for the
# bench line's roofline.traffic (profiles/ncu_traffic.json). Each bench
# command first runs without ncu; ncu then captures consecutive
# pass-kernel launches (fft_pass4_kernel / fft_pass_kernel) inside the step loop.
#   ./paper_1808_06357_b200/tools/ncu_traffic.sh r1g
#   python paper_1808_06357_b200/tools/ncu_traffic.py r1g   (here)
set -u
cd "$(dirname "$0")/../.."
T=gpurun_out/$1
mkdir -p "$T"
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
run() {  # name, skip, count, bench args...
  local name=$1 skip=$2 count=$3; shift 3
  python bench.py "$@" > "$T/${name}_plain.json" 2> "$T/${name}_plain.err"; local rc=$?
  echo "$name plain rc=$rc" >> "$T/status_traffic.txt"
  if [ "$rc" = 0 ]; then
    ncu --clock-control none -k regex:fft_pass --launch-skip "$skip" --launch-count "$count" \
        --metrics "$M" --csv python bench.py "$@" > "$T/${name}_traffic.csv" 2> "$T/${name}_traffic.err"
    echo "$name ncu rc=$?" >> "$T/status_traffic.txt"
  fi
}
run C2 10 4 --config C2 --steps 1 --warmup 3 --m 8 --no-cpu
run C3 10 4 --config C3 --steps 1 --warmup 3 --m 8 --no-cpu
run C4 8 20 --config C4 --steps 1 --warmup 1 --m 3 --no-cpu
cat "$T/status_traffic.txt"

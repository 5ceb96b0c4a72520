#!/usr/bin/env bash
# ncu of config 4's pass kernels (demangled-name filter) and of the opt-in
# cluster COL pass in the devtest (C = 4, minBlocks 3 instance).
set -u
cd "$(dirname "$0")/../.."
T=gpurun_out/$1
mkdir -p "$T"
timeout 600 ./paper_1808_06357_b200/csrc/build/fft_devtest cluster > "$T/devtest_cluster2.txt" 2>&1; rc=$?; echo "devtest rc=$rc" >> "$T/status_ncu2.txt"
if [ "$rc" = 0 ]; then
  ncu --set full --import-source on --clock-control none -k regex:cluster_col_kernel --launch-skip 65 --launch-count 1 \
      -o "$T/prof_cluster" ./paper_1808_06357_b200/csrc/build/fft_devtest cluster > "$T/ncu_cluster.log" 2>&1; echo "ncu cluster rc=$?" >> "$T/status_ncu2.txt"
fi
B4="python bench.py --config C4 --steps 1 --warmup 1 --m 2 --no-cpu"
ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section Occupancy --section LaunchStats \
    --section WarpStateStats --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none --kernel-name-base demangled -k 'regex:fft_pass_kernel<(1, 486|0, 2048|1, 2160)' \
    --launch-skip 6 --launch-count 4 -o "$T/prof_c4" $B4 > "$T/ncu_c4.log" 2>&1; echo "ncu c4 rc=$?" >> "$T/status_ncu2.txt"
cat "$T/status_ncu2.txt"

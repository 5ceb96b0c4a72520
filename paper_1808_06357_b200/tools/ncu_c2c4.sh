#!/usr/bin/env bash
# ncu evidence for the config-2 and config-4 pass kernels (GPU box, one call):
# the bench command first runs without ncu, then the same command under ncu.
#   ./paper_1808_06357_b200/tools/ncu_c2c4.sh r1e
set -u
cd "$(dirname "$0")/../.."
T=gpurun_out/$1
mkdir -p "$T"
B2="python bench.py --config C2 --steps 1 --warmup 3 --m 8 --no-cpu"
$B2 > "$T/c2_plain.json" 2> "$T/c2_plain.err"; rc=$?; echo "c2 plain rc=$rc" >> "$T/status_ncu.txt"
if [ "$rc" = 0 ]; then
  ncu --set full --import-source on --clock-control none -k regex:fft_pass_kernel --launch-skip 8 --launch-count 2 \
      -o "$T/prof_c2" $B2 > "$T/ncu_c2.log" 2>&1; echo "ncu c2 rc=$?" >> "$T/status_ncu.txt"
fi
B4="python bench.py --config C4 --steps 1 --warmup 1 --m 2 --no-cpu"
$B4 > "$T/c4_plain.json" 2> "$T/c4_plain.err"; rc=$?; echo "c4 plain rc=$rc" >> "$T/status_ncu.txt"
if [ "$rc" = 0 ]; then
  ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section Occupancy --section LaunchStats \
      --section WarpStateStats --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k 'regex:fft_pass_kernel<(1, 486|0, 2048|1, 2160)' --launch-skip 6 --launch-count 4 \
      -o "$T/prof_c4" $B4 > "$T/ncu_c4.log" 2>&1; echo "ncu c4 rc=$?" >> "$T/status_ncu.txt"
fi
bash paper_1808_06357_b200/tools/c4_geom_sweep.sh 2160x486x2048 1080x486x4096 > "$T/c4sweep3.txt" 2>&1
cat "$T/status_ncu.txt" "$T/c4sweep3.txt"

#!/usr/bin/env bash
# All GPU artefacts of a round into gpurun_out/<tag>/ (GPU box, one call):
# tests, smoke, bench lines (C1 headline + reference arm, C2, C3, C4), then
# the ncu launch list / full capture / steady-state DRAM of the SAME bench
# command, each only after that command exited 0 without ncu.
#   ./paper_1808_06357_b200/tools/round_artifacts.sh r1b
#   python paper_1808_06357_b200/tools/summarize_profiles.py r1b   (here)
set -u
cd "$(dirname "$0")/../.."
T=gpurun_out/$1
mkdir -p "$T"
python -m pytest tests -m gpu -q > "$T/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$T/status.txt"
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > "$T/smoke.log" 2>&1; echo "smoke rc=$?" >> "$T/status.txt"
python bench.py --steps 5 --warmup 3 > "$T/bench_C1.json" 2> "$T/bench_C1.err"; rc=$?; echo "bench C1 rc=$rc" >> "$T/status.txt"
python bench.py --impl reference --steps 3 --warmup 1 > "$T/bench_reference_C1.json" 2> "$T/bench_reference_C1.err"; echo "reference rc=$?" >> "$T/status.txt"
python bench.py --config C2 --steps 3 --warmup 3 --no-cpu > "$T/bench_C2.json" 2> "$T/bench_C2.err"; echo "bench C2 rc=$?" >> "$T/status.txt"
python bench.py --config C3 --steps 3 --warmup 3 --no-cpu > "$T/bench_C3.json" 2> "$T/bench_C3.err"; echo "bench C3 rc=$?" >> "$T/status.txt"
python bench.py --config C4 --steps 2 --warmup 3 > "$T/bench_C4.json" 2> "$T/bench_C4.err"; echo "bench C4 rc=$?" >> "$T/status.txt"
if [ "$rc" = 0 ]; then
  B="python bench.py --steps 1 --warmup 3 --no-cpu"
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv $B > "$T/launches.csv" 2> "$T/launches.err"
  echo "ncu launches rc=$?" >> "$T/status.txt"
  ncu --set full --import-source on --clock-control none -k regex:fft_pass_kernel --launch-skip 60 --launch-count 2 \
      -o "$T/prof_c1" $B > "$T/ncu_full.log" 2>&1
  echo "ncu full rc=$?" >> "$T/status.txt"
  ncu --cache-control none --clock-control none -k regex:fft_pass_kernel --launch-skip 60 --launch-count 4 \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv $B > "$T/ncu_steady.csv" 2> "$T/ncu_steady.err"
  echo "ncu steady rc=$?" >> "$T/status.txt"
fi
cat "$T/status.txt"

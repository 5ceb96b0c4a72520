#!/usr/bin/env bash
# All GPU artefacts of a round into gpurun_out/<tag>/ (GPU box, one call):
# tests, smoke, the default bench line (config 3) + reference arm, bench lines
# of the other configs, then the ncu launch list / full capture of the SAME
# bench command (each only after that command exited 0 without ncu) and the
# DRAM traffic per pass launch (ncu_traffic.sh).
#   ./paper_1808_06357_b200/tools/round_artifacts.sh r2
#   python paper_1808_06357_b200/tools/summarize_profiles.py r2   (here)
set -u
cd "$(dirname "$0")/../.."
T=gpurun_out/$1
mkdir -p "$T"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > "$T/gpu.txt"
python -m pytest tests -m gpu -q > "$T/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$T/status.txt"
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > "$T/smoke.log" 2>&1; echo "smoke rc=$?" >> "$T/status.txt"
python bench.py --steps 5 --warmup 3 > "$T/bench_C3.json" 2> "$T/bench_C3.err"; rc=$?; echo "bench C3 rc=$rc" >> "$T/status.txt"
python bench.py --impl reference --steps 3 --warmup 1 > "$T/bench_reference_C3.json" 2> "$T/bench_reference_C3.err"; echo "reference rc=$?" >> "$T/status.txt"
python bench.py --config C1 --steps 5 --warmup 3 --no-cpu > "$T/bench_C1.json" 2> "$T/bench_C1.err"; echo "bench C1 rc=$?" >> "$T/status.txt"
python bench.py --config C2 --steps 3 --warmup 3 --no-cpu > "$T/bench_C2.json" 2> "$T/bench_C2.err"; echo "bench C2 rc=$?" >> "$T/status.txt"
python bench.py --config C4 --steps 2 --warmup 3 --no-cpu > "$T/bench_C4.json" 2> "$T/bench_C4.err"; echo "bench C4 rc=$?" >> "$T/status.txt"
if [ "$rc" = 0 ]; then
  B="python bench.py --m 4 --steps 1 --warmup 3 --no-cpu"
  $B > "$T/plain.log" 2>&1 && {
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fft_pass -c 400 --csv --log-file "$T/launches.csv" $B > "$T/launches.log" 2>&1
  echo "ncu launches rc=$?" >> "$T/status.txt"
  ncu --set full --import-source on --clock-control none -k regex:fft_pass --launch-skip 12 --launch-count 2 \
      -f -o "$T/prof_c3" $B > "$T/ncu_full.log" 2>&1
  echo "ncu full rc=$?" >> "$T/status.txt"
  }
fi
./paper_1808_06357_b200/tools/ncu_traffic.sh "$1" > "$T/traffic.log" 2>&1
cat "$T/status.txt"

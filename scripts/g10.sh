# one compute-sanitizer tool per gpurun call (B200_PROFILING.md)
mkdir -p gpurun_out/r2san
TOOL=${1:-racecheck}
timeout 1500 compute-sanitizer --tool $TOOL --error-exitcode 9 --print-limit 50 python tests/sanitize_case.py > gpurun_out/r2san/$TOOL.log 2>&1
echo "$TOOL rc=$?" | tee -a gpurun_out/r2san/$TOOL.log
tail -5 gpurun_out/r2san/$TOOL.log

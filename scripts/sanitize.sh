# one compute-sanitizer tool per gpurun call: scripts/sanitize.sh racecheck
TOOL=${1:-racecheck}
LATTDSE_SANITIZE=$TOOL timeout 3300 python -m pytest tests/test_gpu_sanitizer.py -m gpu -q -x 2>&1 | tail -5
tail -12 gpurun_out/sanitizer_$TOOL.log

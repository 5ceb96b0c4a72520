set -u
mkdir -p gpurun_out/c4ab
timeout 900 python -m pytest tests -m gpu -q -x -k "three_level or config4" > gpurun_out/c4ab/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c4ab/status.txt
for ch in 0 -1 2; do
  LATTDSE_ROW_CHUNK=$ch timeout 900 python bench.py --config C4 --steps 1 --warmup 3 --m 8 --no-cpu > gpurun_out/c4ab/bench_chunk$ch.json 2> gpurun_out/c4ab/bench_chunk$ch.err; echo "bench $ch rc=$?" >> gpurun_out/c4ab/status.txt
done
cat gpurun_out/c4ab/status.txt

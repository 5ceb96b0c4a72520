set -x
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
./bin_tmp/fp64_peak > gpurun_out/r2a/fp64_peak.txt 2>&1; cat gpurun_out/r2a/fp64_peak.txt
python bench.py --config C3 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2a/bench_c3.json 2> gpurun_out/r2a/bench_c3.err; tail -c 3000 gpurun_out/r2a/bench_c3.json
python bench.py --config C3 --m 2 --steps 1 --warmup 3 --no-cpu > gpurun_out/r2a/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:fft_pass_kernel<1, 1080, 2, 384, 0|fft_pass_kernel<0, 486" -c 4 -o gpurun_out/r2a/c3 python bench.py --config C3 --m 2 --steps 1 --warmup 3 --no-cpu > gpurun_out/r2a/ncu.log 2>&1
tail -5 gpurun_out/r2a/ncu.log

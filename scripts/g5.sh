mkdir -p gpurun_out/r2e
export LATTDSE_PASS3=0
python bench.py --config C3 --m 2 --steps 1 --warmup 3 --no-cpu > gpurun_out/r2e/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:fft_pass_kernel<\(int\)1, \(int\)1080, \(int\)2, \(int\)288, \(int\)0|fft_pass_kernel<\(int\)0, \(int\)486, \(int\)1, \(int\)96, \(int\)0' \
  -c 5 -o gpurun_out/r2e/c3new python bench.py --config C3 --m 2 --steps 1 --warmup 3 --no-cpu > gpurun_out/r2e/ncu.log 2>&1
tail -2 gpurun_out/r2e/ncu.log

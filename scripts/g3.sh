mkdir -p gpurun_out/r2c
export LATTDSE_PASS3=0
python bench.py --config C3 --m 2 --steps 1 --warmup 3 --no-cpu > gpurun_out/r2c/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:fft_pass_kernel<\(int\)1, \(int\)1080, \(int\)2, \(int\)384, \(int\)0|fft_pass_kernel<\(int\)0, \(int\)486, \(int\)1, \(int\)96, \(int\)0' \
  -c 2 -o gpurun_out/r2c/c3v1 python bench.py --config C3 --m 2 --steps 1 --warmup 3 --no-cpu > gpurun_out/r2c/ncu1.log 2>&1
tail -3 gpurun_out/r2c/ncu1.log
export LATTDSE_PASS3=1
python bench.py --config C3 --m 2 --steps 1 --warmup 3 --no-cpu > gpurun_out/r2c/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:fft_pass3_kernel' -c 2 -o gpurun_out/r2c/c3v3 python bench.py --config C3 --m 2 --steps 1 --warmup 3 --no-cpu > gpurun_out/r2c/ncu3.log 2>&1
tail -3 gpurun_out/r2c/ncu3.log

mkdir -p gpurun_out/r2f
export LATTDSE_PASS3=0
for G in 1080x486 486x1080 729x720 720x729; do
  LATTDSE_GEOM=$G python bench.py --config C3 --m 64 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2f/c3_$G.json 2> gpurun_out/r2f/c3_$G.err
  python -c "import json;d=json.load(open('gpurun_out/r2f/c3_$G.json'));print('C3 $G', d['us_per_strang_step'], {k:(round(v['ms'],3),round(v['frac'],3)) for k,v in d['roofline']['passes'].items()})"
done
LATTDSE_GEOM=486x1080 python bench.py --config C3 --m 2 --steps 1 --warmup 3 --no-cpu > gpurun_out/r2f/plain.log 2>&1 && \
LATTDSE_GEOM=486x1080 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:fft_pass_kernel<\(int\)1, \(int\)486, \(int\)4, .*\(int\)0, \(int\)1|fft_pass_kernel<\(int\)0, \(int\)1080, \(int\)1, .*\(int\)0, \(int\)-1' \
  -c 4 -o gpurun_out/r2f/c3swap python bench.py --config C3 --m 2 --steps 1 --warmup 3 --no-cpu > gpurun_out/r2f/ncu.log 2>&1
tail -2 gpurun_out/r2f/ncu.log

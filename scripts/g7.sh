mkdir -p gpurun_out/r2g
export LATTDSE_PASS3=0
cp paper_1808_06357_b200/liblattdse_b200.so /tmp/lib_A.so
for V in A B C D F; do
  if [ $V = A ]; then cp /tmp/lib_A.so paper_1808_06357_b200/liblattdse_b200.so; else xz -dc bin_tmp/var_$V.so.xz > paper_1808_06357_b200/liblattdse_b200.so; fi
  for G in 486x1080 1080x486; do
    LATTDSE_GEOM=$G python bench.py --config C3 --m 64 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2g/c3_${V}_$G.json 2> gpurun_out/r2g/c3_${V}_$G.err
    python -c "import json;d=json.load(open('gpurun_out/r2g/c3_${V}_$G.json'));print('$V $G', round(d['us_per_strang_step'],1), {k:(round(v['ms'],3),round(v['frac'],3)) for k,v in d['roofline']['passes'].items()})"
  done
done
cp /tmp/lib_A.so paper_1808_06357_b200/liblattdse_b200.so

T=gpurun_out/r2d; mkdir -p $T
for P in 1 0; do
  LATTDSE_L2_PERSIST=$P python bench.py --config C3 --m 64 --steps 3 --warmup 3 --no-cpu > $T/C3_persist$P.json 2> $T/err
  python -c "import json;d=json.load(open('$T/C3_persist$P.json'));print('C3 persist=$P', round(d['us_per_strang_step'],1), {k:(round(v['ms'],3),round(v['frac'],3)) for k,v in d['roofline']['passes'].items()}, d['clocks'])"
done

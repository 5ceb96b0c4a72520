T=gpurun_out/r2g; mkdir -p $T
for G in 8 10 12 16 32 512; do
  LATTDSE_GROUP=$G python bench.py --config C3 --m 64 --steps 3 --warmup 3 --no-cpu > $T/C3_g$G.json 2> $T/err
  python -c "import json;d=json.load(open('$T/C3_g$G.json'));print('C3 group=$G', round(d['us_per_strang_step'],1), d['clocks']['sm_mhz'], d['solver']['group'])"
done

set -u
T=gpurun_out/${TAG:-r2i}
mkdir -p $T
python -m pytest tests/test_gpu_config4.py tests/test_gpu_parity.py -x -q -k "config4 or c4r or three_level or sharded or C4" > $T/pytest_c4.log 2>&1; tail -4 $T/pytest_c4.log
for P in 1 0; do
  LATTDSE_PASS4=$P python bench.py --config C4 --m 16 --steps 2 --warmup 3 --no-cpu > $T/C4_p$P.json 2> $T/C4_p$P.err
  python -c "import json;d=json.load(open('$T/C4_p$P.json'));print('C4 pass4=$P', round(d['us_per_strang_step'],1), {k:(round(v['ms'],3),round(v['frac'],3)) for k,v in d['roofline']['passes'].items()}, round(d['roofline']['step']['frac'],3))"
done

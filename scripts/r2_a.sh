set -u
T=gpurun_out/r2a
mkdir -p $T
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullrun.py -x -q > $T/pytest_parity.log 2>&1; tail -3 $T/pytest_parity.log
for P in 1 0; do
for C in C3:64 C1:256 C2:64; do
  c=${C%%:*}; m=${C##*:}
  LATTDSE_PASS4=$P python bench.py --config $c --m $m --steps 3 --warmup 3 --no-cpu > $T/${c}_p$P.json 2> $T/${c}_p$P.err
  python -c "import json;d=json.load(open('$T/${c}_p$P.json'));print('$c pass4=$P', round(d['us_per_strang_step'],1), {k:(round(v['ms'],3),round(v['frac'],3)) for k,v in d['roofline']['passes'].items()}, d['solver']['pass_kernel'])"
done
done

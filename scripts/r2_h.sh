set -u
T=gpurun_out/${TAG:-r2h}
mkdir -p $T
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullrun.py tests/test_gpu_pass4.py tests/test_gpu_config4.py -x -q > $T/pytest_parity.log 2>&1; tail -3 $T/pytest_parity.log
for C in C2:64 C4:16 C1:256 C3:64; do
  c=${C%%:*}; m=${C##*:}
  python bench.py --config $c --m $m --steps 3 --warmup 3 --no-cpu > $T/${c}.json 2> $T/${c}.err
  python -c "import json;d=json.load(open('$T/${c}.json'));print('$c', round(d['us_per_strang_step'],1), {k:(round(v['ms'],3),round(v['frac'],3)) for k,v in d['roofline']['passes'].items()}, round(d['roofline']['step']['frac'],3), d['solver']['pass_kernel'])"
done

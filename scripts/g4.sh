mkdir -p gpurun_out/r2d
for P in 0 1; do
  LATTDSE_PASS3=$P python bench.py --config C3 --m 64 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2d/c3_p$P.json 2> gpurun_out/r2d/c3_p$P.err
  python -c "import json;d=json.load(open('gpurun_out/r2d/c3_p$P.json'));print('C3 pass3=$P', d['us_per_strang_step'], d['roofline']['passes'])"
  LATTDSE_PASS3=$P python bench.py --config C1 --m 256 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2d/c1_p$P.json 2> gpurun_out/r2d/c1_p$P.err
  python -c "import json;d=json.load(open('gpurun_out/r2d/c1_p$P.json'));print('C1 pass3=$P', d['us_per_strang_step'], d['roofline']['passes'])"
done
python -m pytest tests/ -m gpu -x -q > gpurun_out/r2d/pytest.log 2>&1; tail -5 gpurun_out/r2d/pytest.log

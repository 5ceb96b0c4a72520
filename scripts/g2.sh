# pass3 A/B on C3 and C1 + parity subset
mkdir -p gpurun_out/r2b
python -m pytest tests/test_gpu_parity.py -x -q -k "rank1_small or config0 or rank2" > gpurun_out/r2b/pytest.log 2>&1; tail -3 gpurun_out/r2b/pytest.log
for P in 1 0; do
  LATTDSE_PASS3=$P python bench.py --config C3 --m 64 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2b/c3_p$P.json 2> gpurun_out/r2b/c3_p$P.err
  python -c "import json;d=json.load(open('gpurun_out/r2b/c3_p$P.json'));print('C3 pass3=$P', d['us_per_strang_step'], d['roofline']['pass_ms'])"
  LATTDSE_PASS3=$P python bench.py --config C1 --m 256 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2b/c1_p$P.json 2> gpurun_out/r2b/c1_p$P.err
  python -c "import json;d=json.load(open('gpurun_out/r2b/c1_p$P.json'));print('C1 pass3=$P', d['us_per_strang_step'], d['roofline']['pass_ms'])"
done
for PR in 2 1; do
  LATTDSE_TMA_PROMO=$PR python bench.py --config C3 --m 64 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2b/c3_promo$PR.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/r2b/c3_promo$PR.json'));print('C3 promo=$PR', d['us_per_strang_step'], d['roofline']['pass_ms'])"
done

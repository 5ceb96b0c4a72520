mkdir -p gpurun_out/r2i
python bench.py --config C3 --m 64 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2i/c3.json 2> gpurun_out/r2i/c3.err
python -c "import json;d=json.load(open('gpurun_out/r2i/c3.json'));print('C3', round(d['us_per_strang_step'],1), {k:(round(v['ms'],3),round(v['frac'],3)) for k,v in d['roofline']['passes'].items()})"
python bench.py --config C1 --m 256 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2i/c1.json 2> gpurun_out/r2i/c1.err
python -c "import json;d=json.load(open('gpurun_out/r2i/c1.json'));print('C1', round(d['us_per_strang_step'],1), {k:(round(v['ms'],3),round(v['frac'],3)) for k,v in d['roofline']['passes'].items()})"
python bench.py --config C2 --m 64 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2i/c2.json 2> gpurun_out/r2i/c2.err
python -c "import json;d=json.load(open('gpurun_out/r2i/c2.json'));print('C2', round(d['us_per_strang_step'],1), {k:(round(v['ms'],3),round(v['frac'],3)) for k,v in d['roofline']['passes'].items()})"
python -m pytest tests/ -m gpu -q -x --deselect tests/test_gpu_config4.py > gpurun_out/r2i/pytest.log 2>&1; tail -8 gpurun_out/r2i/pytest.log

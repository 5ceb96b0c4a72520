mkdir -p gpurun_out/r2h
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python bench.py > gpurun_out/r2h/bench_default.json 2> gpurun_out/r2h/bench_default.err; tail -c 2500 gpurun_out/r2h/bench_default.json
python bench.py --impl reference > gpurun_out/r2h/bench_reference.json 2> gpurun_out/r2h/bench_reference.err; tail -c 600 gpurun_out/r2h/bench_reference.json
python -m pytest tests/ -m gpu -q > gpurun_out/r2h/pytest.log 2>&1; tail -15 gpurun_out/r2h/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h/smoke.log 2>&1; tail -2 gpurun_out/r2h/smoke.log

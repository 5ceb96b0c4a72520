# Round-2 baseline on the restored tree: GPU tests, smoke, default bench (C3), reference arm,
# ncu launch list + full capture of the two C3 step kernels.
set -u
T=gpurun_out/r2base
mkdir -p $T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $T/gpu.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $T/smoke.log 2>&1; echo "smoke rc=$?" >> $T/status.txt
python bench.py --steps 3 --warmup 3 > $T/bench_C3.json 2> $T/bench_C3.err; rc=$?; echo "bench C3 rc=$rc" >> $T/status.txt
python -c "import json;d=json.load(open('$T/bench_C3.json'));print('C3', d['value'], d['e2e']['value'], round(d['us_per_strang_step'],1), {k:(round(v['ms'],3),round(v['frac'],3)) for k,v in d['roofline']['passes'].items()}, d['solver'])"
python bench.py --impl reference --steps 2 --warmup 1 > $T/bench_reference.json 2> $T/bench_reference.err; echo "reference rc=$?" >> $T/status.txt
B="python bench.py --m 4 --steps 1 --warmup 3 --no-cpu"
$B > $T/plain.log 2>&1 && {
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $T/launches.csv $B > $T/launches.log 2>&1
echo "ncu launches rc=$?" >> $T/status.txt
ncu --set full --import-source on --clock-control none -k regex:fft_pass_kernel --launch-skip 12 --launch-count 2 -o $T/prof_c3 $B > $T/ncu_full.log 2>&1
echo "ncu full rc=$?" >> $T/status.txt
}
timeout 2400 python -m pytest tests -m gpu -q -x > $T/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $T/status.txt
tail -5 $T/pytest_gpu.log
cat $T/status.txt

set -u
T=gpurun_out/r2p3
mkdir -p $T
./bin_tmp/fp64_peak > $T/fp64_peak.txt 2>&1; cat $T/fp64_peak.txt
for P in 0 1; do
  LATTDSE_PASS3=$P python bench.py --config C3 --m 64 --steps 3 --warmup 3 --no-cpu > $T/c3_p$P.json 2> $T/c3_p$P.err
  python -c "import json;d=json.load(open('$T/c3_p$P.json'));print('C3 pass3=$P', round(d['us_per_strang_step'],1), {k:(round(v['ms'],3),round(v['frac'],3)) for k,v in d['roofline']['passes'].items()})"
done
LATTDSE_PASS3=1 ncu --set full --import-source on --clock-control none -k regex:fft_pass3_kernel --launch-skip 12 --launch-count 2 -o $T/prof_p3 python bench.py --m 4 --steps 1 --warmup 3 --no-cpu > $T/ncu_full.log 2>&1
tail -3 $T/ncu_full.log

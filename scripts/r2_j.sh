T=gpurun_out/r2j; mkdir -p $T
cp paper_1808_06357_b200/liblattdse_b200.so /tmp/lib_main.so
for V in main B8; do
  if [ $V = B8 ]; then cp bin_tmp/varB8/liblattdse_b200.so paper_1808_06357_b200/liblattdse_b200.so; fi
  python bench.py --config C4 --m 16 --steps 2 --warmup 3 --no-cpu > $T/C4_$V.json 2> $T/C4_$V.err
  python -c "import json;d=json.load(open('$T/C4_$V.json'));print('C4 $V', round(d['us_per_strang_step'],1), {k:(round(v['ms'],3),round(v['frac'],3)) for k,v in d['roofline']['passes'].items()})"
  python bench.py --config C3 --m 64 --steps 3 --warmup 3 --no-cpu > $T/C3_$V.json 2> $T/C3_$V.err
  python -c "import json;d=json.load(open('$T/C3_$V.json'));print('C3 $V', round(d['us_per_strang_step'],1), {k:(round(v['ms'],3),round(v['frac'],3)) for k,v in d['roofline']['passes'].items()})"
done
cp /tmp/lib_main.so paper_1808_06357_b200/liblattdse_b200.so

# geometry sweep with the lean kernels: every split of M among the compiled lengths
T=gpurun_out/r2geom; mkdir -p $T
for G in 486x1080 1080x486 729x720 720x729 810x648 648x810 972x540 540x972 405x1296 1296x405 432x1215 1215x432 324x1620 1620x324 243x2160 2160x243; do
  LATTDSE_GEOM=$G python bench.py --config C3 --m 32 --steps 2 --warmup 3 --no-cpu > $T/c3_$G.json 2> $T/c3_$G.err
  python -c "import json;d=json.load(open('$T/c3_$G.json'));print('C3 $G', d['solver']['M1'], d['solver']['M2'], round(d['us_per_strang_step'],1), {k:(round(v['ms'],3),round(v['frac'],3)) for k,v in d['roofline']['passes'].items()})" 2>/dev/null || echo "C3 $G failed"
done
for G in 1296x1620 1620x1296 1080x1944 1944x1080 972x2160 2160x972 1215x1728 1728x1215 1458x1440 1440x1458 720x2916 810x2592; do
  LATTDSE_GEOM=$G python bench.py --config C1 --m 256 --steps 2 --warmup 3 --no-cpu > $T/c1_$G.json 2> $T/c1_$G.err
  python -c "import json;d=json.load(open('$T/c1_$G.json'));print('C1 $G', d['solver']['M1'], d['solver']['M2'], round(d['us_per_strang_step'],1), {k:(round(v['ms'],3),round(v['frac'],3)) for k,v in d['roofline']['passes'].items()})" 2>/dev/null || echo "C1 $G failed"
done

set -u
T=gpurun_out/${TAG:-r2b}
mkdir -p $T
B="python bench.py --config ${CFG:-C3} --m 4 --steps 1 --warmup 3 --no-cpu"
$B > $T/plain.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:fft_pass --launch-skip ${SKIP:-12} --launch-count 2 -f -o $T/prof $B > $T/ncu_full.log 2>&1
tail -2 $T/ncu_full.log

# config-4 DRAM traffic capture alone (two step COL launches: m = 3)
T=gpurun_out/r2; mkdir -p $T
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
A="--config C4 --steps 1 --warmup 1 --m 3 --no-cpu"
python bench.py $A > $T/C4_plain.json 2> $T/C4_plain.err && \
ncu --clock-control none -k regex:fft_pass --launch-skip 8 --launch-count 20 --metrics $M --csv python bench.py $A > $T/C4_traffic.csv 2> $T/C4_traffic.err
echo "C4 rc=$?"

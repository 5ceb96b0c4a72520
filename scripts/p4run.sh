# p4run.sh: run every bin_tmp/p4_* variant; ncu the first two cases of p4_a
mkdir -p gpurun_out/p4
for f in bin_tmp/p4_*; do case $f in *.ptxas) continue;; esac; echo "== $f"; $f ${BATCH:-64} 2>&1 | grep -E "TIME|MISMATCH" ; done | tee gpurun_out/p4/run.txt
if [ -n "${NCU:-}" ]; then
for c in $NCU; do
ncu --set full --import-source on --clock-control none -k regex:fft_pass4_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/p4/prof_${NCUBIN:-p4_a}_$c -f bin_tmp/${NCUBIN:-p4_a} 16 $c > gpurun_out/p4/ncu_$c.log 2>&1; tail -2 gpurun_out/p4/ncu_$c.log
done
fi

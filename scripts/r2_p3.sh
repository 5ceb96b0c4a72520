# FP64 issue rate and shared-memory bandwidth of the board (tools/fp64_peak.cu,
# built to bin_tmp/fp64_peak): the in-SM co-limits of the pass kernels
set -u
T=gpurun_out/r2p3
mkdir -p $T
./bin_tmp/fp64_peak > $T/fp64_peak.txt 2>&1; cat $T/fp64_peak.txt

#!/bin/bash
# build_variant.sh NAME "L,r0,r1,r2,r3" "L,r0,r1,r2,r3": a copy of the library
# whose pass kernels for those two lengths use the given radix plans
# (fft_core.cuh LATTDSE_PLAN_X/Y), into bin_tmp/var_NAME/liblattdse_b200.so
set -e
NAME=$1; PX=$2; PY=$3
cd /root/repo/paper_1808_06357_b200/csrc
OUT=/root/repo/bin_tmp/var_$NAME; mkdir -p $OUT/obj
LX=${PX%%,*}; LY=${PY%%,*}
printf '#define LATTDSE_PLAN_X %s\n#define LATTDSE_PLAN_Y %s\n' "$PX" "$PY" > $OUT/plan.h
for L in $LX $LY; do
  nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo --expt-relaxed-constexpr -diag-suppress 20014 \
    -Xcompiler -fPIC,-fopenmp -I/root/repo/include -Ihost -Icuda -include $OUT/plan.h \
    -c cuda/inst/pass_L$L.cu -o $OUT/obj/pass_L$L.o
done
OBJS=$(ls build/host/*.o build/cuda/*.o build/cuda/inst/*.o | grep -v "pass_L$LX.o\|pass_L$LY.o\|cluster_col")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $OUT/liblattdse_b200.so $OBJS $OUT/obj/*.o -Xcompiler -fopenmp -lgomp
echo built $OUT

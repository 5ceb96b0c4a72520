#!/bin/bash
# p4build.sh NAME "PLANX" "PLANY" 'CASES': pass4 devtest variant bin_tmp/p4_NAME
# PLANX/PLANY: "L,r0,r1,r2,r3" radix plan overrides ("" = none); CASES: CASE((run<...>(...))) list ("" = default)
set -e
NAME=$1; PX=$2; PY=$3; CASES=$4; EXTRA=${5:-}
cd /root/repo/paper_1808_06357_b200/csrc
H=/root/repo/bin_tmp/p4_$NAME.h
: > $H
[ -n "$PX" ] && echo "#define LATTDSE_PLAN_X $PX" >> $H
[ -n "$PY" ] && echo "#define LATTDSE_PLAN_Y $PY" >> $H
[ -n "$CASES" ] && echo "#define P4_CASES $CASES" >> $H
[ -n "$EXTRA" ] && echo "$EXTRA" >> $H
nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo --expt-relaxed-constexpr -diag-suppress 20014 -Xptxas -v -Icuda -I../../include -include $H cuda/fft_pass4_devtest.cu -o /root/repo/bin_tmp/p4_$NAME 2> /root/repo/bin_tmp/p4_$NAME.ptxas || { grep -m5 error /root/repo/bin_tmp/p4_$NAME.ptxas; exit 1; }
python3 - <<PY
import re
t=open('/root/repo/bin_tmp/p4_$NAME.ptxas').read()
for m in re.finditer(r"Function properties for (\S+)\n\s+(\d+) bytes stack frame, (\d+) bytes spill stores.*\n.*Used (\d+) registers",t):
    n=m.group(1)
    if 'pass4' in n: print('$NAME', re.sub(r'_ZN11lattdse_dev16fft_pass4_kernelI','',n)[:60], 'regs',m.group(4),'spill',m.group(3))
PY

#!/bin/bash
# ncu --set full capture of chosen kernels in one C5 bench step.
# usage: tools/gpu_ncu.sh TAG REGEX [SKIP] [COUNT]
set -u
O=gpurun_out
T=${1:-x}; RX=${2:-solve_kernel}; S=${3:-40}; C=${4:-3}
make -s all >/dev/null 2>&1 || { echo build failed; exit 1; }
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s $S -c $C -f -o $O/prof_$T $CMD > $O/ncu_$T.log 2>&1; echo rc=$? >> $O/ncu_$T.log

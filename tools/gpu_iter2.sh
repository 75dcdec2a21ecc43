#!/bin/bash
# iteration run: full gpu test suite, C5 bench, ncu of the projection + SpMM kernels
set -u
O=gpurun_out
T=${1:-x}
make -s all >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q -p no:hypothesispytest > $O/pytest_$T.log 2>&1; echo rc=$? >> $O/pytest_$T.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$T.log 2>&1; echo rc=$? >> $O/bench_$T.log
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --kernel-name-base function -k regex:"^(partial_kernel|recon_kernel|spmm_kernel)$" -s 6 -c 6 -o $O/prof_proj_$T $CMD > $O/ncu_proj_$T.log 2>&1
echo rc=$? >> $O/ncu_proj_$T.log

#!/bin/bash
# gpu tests, F4 bench, ncu of projection kernels (C5) and the bilateral sweep (F4)
set -u
O=gpurun_out
T=${1:-x}
make -s all >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -p no:hypothesispytest > $O/pytest_$T.log 2>&1; echo rc=$? >> $O/pytest_$T.log
timeout 600 python bench.py --config F4 --steps 3 --warmup 3 > $O/bench_f4_$T.log 2>&1; echo rc=$? >> $O/bench_f4_$T.log
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --kernel-name-base function -k regex:"^(partial_kernel|recon_kernel)$" -s 40 -c 4 -o $O/prof_proj_$T $CMD > $O/ncu_proj_$T.log 2>&1
echo rc=$? >> $O/ncu_proj_$T.log
F4="python bench.py --config F4 --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --kernel-name-base function -k regex:"^(bilateral_kernel|vertex_update_kernel)$" -s 2 -c 2 -o $O/prof_fine_$T $F4 > $O/ncu_fine_$T.log 2>&1
echo rc=$? >> $O/ncu_fine_$T.log

#!/bin/bash
# F3 frames path: gpu tests + F3 bench; ncu of the HBM-side kernels (SpMM, projection) in the C5 step
set -u
O=gpurun_out
T=${1:-r01d}
make -s >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_frames.py -x -q -p no:hypothesispytest > $O/pytest_frames_$T.log 2>&1; echo rc=$? >> $O/pytest_frames_$T.log
timeout 900 python bench.py --config F3 --steps 3 --warmup 3 > $O/bench_f3_$T.log 2>&1; echo rc=$? >> $O/bench_f3_$T.log
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none -k regex:"spmm_kernel|partial_kernel|recon_kernel" -s 200 -c 6 -o $O/prof_hbm_$T $CMD > $O/ncu_hbm_$T.log 2>&1
echo ncu_hbm rc=$? >> $O/ncu_hbm_$T.log
F3="python bench.py --config F3 --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_f3_$T.csv $F3 > $O/ncu_list_f3_$T.log 2>&1
echo ncu_list rc=$? >> $O/ncu_list_f3_$T.log

#!/bin/bash
# Round evidence: GPU tests, smoke, default bench (+CPU baseline), reference arm,
# C1-C4 + F3/F4 bench lines, small-batch sweep, one-step launch list, ncu captures.
set -u
O=gpurun_out
T=${1:-ev}
make -s all >/dev/null 2>&1 || { echo build failed; exit 1; }
nproc > $O/host_$T.txt; lscpu >> $O/host_$T.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:hypothesispytest > $O/pytest_$T.log 2>&1; echo rc=$? >> $O/pytest_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$T.log 2>&1; echo rc=$? >> $O/smoke_$T.log
timeout 900 python bench.py > $O/bench_$T.log 2>&1; echo rc=$? >> $O/bench_$T.log
timeout 900 python bench.py --impl reference > $O/bench_ref_$T.log 2>&1; echo rc=$? >> $O/bench_ref_$T.log
for C in C1 C2 C3; do timeout 600 python bench.py --config $C --steps 5 --warmup 3 > $O/bench_${C}_$T.log 2>&1; echo rc=$? >> $O/bench_${C}_$T.log; done
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_C4_$T.log 2>&1; echo rc=$? >> $O/bench_C4_$T.log
timeout 600 python bench.py --config F3 --steps 3 --warmup 3 > $O/bench_F3_$T.log 2>&1; echo rc=$? >> $O/bench_F3_$T.log
timeout 600 python bench.py --config F4 --steps 20 --warmup 3 > $O/bench_F4_$T.log 2>&1; echo rc=$? >> $O/bench_F4_$T.log
for m in 8 16 32; do timeout 600 python bench.py --meshes $m --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_m${m}_$T.log 2>&1; done
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 6100 -c 6100 --csv --log-file $O/launches_$T.csv $CMD > $O/ncu_list_$T.log 2>&1; echo rc=$? >> $O/ncu_list_$T.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"solve_kernel|recon_mma|partial_kernel|orth_probe|gemm_pipe_kernel|cholx" -s 300 -c 14 -o $O/prof_main_$T $CMD > $O/ncu_full_$T.log 2>&1; echo rc=$? >> $O/ncu_full_$T.log

#!/bin/bash
# one gpurun call: gpu tests, smoke, default bench (with CPU baseline), reference arm,
# ncu launch list of one step, ncu --set full capture of the solve
set -u
O=gpurun_out
T=${1:-r01c}
make -s >/dev/null 2>&1 || { echo build failed; exit 1; }
nproc > $O/host_$T.txt; lscpu >> $O/host_$T.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:hypothesispytest > $O/pytest_$T.log 2>&1; echo rc=$? >> $O/pytest_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$T.log 2>&1; echo rc=$? >> $O/smoke_$T.log
timeout 900 python bench.py > $O/bench_$T.log 2>&1; echo rc=$? >> $O/bench_$T.log
timeout 900 python bench.py --impl reference > $O/bench_ref_$T.log 2>&1; echo rc=$? >> $O/bench_ref_$T.log
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > $O/plain_$T.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 5000 -c 5000 --csv --log-file $O/launches_$T.csv $CMD > $O/ncu_list_$T.log 2>&1
echo ncu_list rc=$? >> $O/plain_$T.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:solve -s 40 -c 2 -o $O/prof_solve_$T $CMD > $O/ncu_full_$T.log 2>&1
echo ncu_full rc=$? >> $O/plain_$T.log

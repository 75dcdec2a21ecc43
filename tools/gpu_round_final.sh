#!/bin/bash
# round-end evidence: gpu tests, smoke, default bench (+CPU baseline), reference arm,
# F3/F4 bench lines, C1-C4 configs, ncu launch list of one C5 step, ncu --set full of the solve
set -u
O=gpurun_out
T=${1:-final}
make -s all tools >/dev/null 2>&1 || { echo build failed; exit 1; }
nproc > $O/host_$T.txt; lscpu >> $O/host_$T.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:hypothesispytest > $O/pytest_$T.log 2>&1; echo rc=$? >> $O/pytest_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$T.log 2>&1; echo rc=$? >> $O/smoke_$T.log
timeout 900 python bench.py > $O/bench_$T.log 2>&1; echo rc=$? >> $O/bench_$T.log
timeout 900 python bench.py --impl reference > $O/bench_ref_$T.log 2>&1; echo rc=$? >> $O/bench_ref_$T.log
timeout 600 python bench.py --config F3 --steps 3 --warmup 3 > $O/bench_f3_$T.log 2>&1; echo rc=$? >> $O/bench_f3_$T.log
timeout 600 python bench.py --config F4 --steps 20 --warmup 3 > $O/bench_f4_$T.log 2>&1; echo rc=$? >> $O/bench_f4_$T.log
timeout 900 python tools/bench_configs.py > $O/configs_$T.log 2>&1; echo rc=$? >> $O/configs_$T.log
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 5000 -c 5000 --csv --log-file $O/launches_$T.csv $CMD > $O/ncu_list_$T.log 2>&1
echo ncu_list rc=$? >> $O/ncu_list_$T.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:solve -s 40 -c 2 -o $O/prof_solve_$T $CMD > $O/ncu_full_$T.log 2>&1
echo ncu_full rc=$? >> $O/ncu_full_$T.log

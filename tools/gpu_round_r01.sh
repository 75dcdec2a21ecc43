#!/bin/bash
# one gpurun call: benches (default, serialized groups, 8-mesh shard) + ncu launch list + ncu full capture of solve
set -u
make -s >/dev/null 2>&1 || { echo build failed; exit 1; }
O=gpurun_out
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_a.log 2>&1; echo rc=$? >> $O/bench_a.log
SMG_GROUPS=1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_g1.log 2>&1; echo rc=$? >> $O/bench_g1.log
python bench.py --meshes 8 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_m8.log 2>&1; echo rc=$? >> $O/bench_m8.log
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 5000 -c 5000 --csv --log-file $O/launches_r01b.csv $CMD > $O/ncu_list.log 2>&1
echo ncu_list rc=$? >> $O/plain.log
$CMD > $O/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:solve -s 40 -c 2 -o $O/prof_solve_r01 $CMD > $O/ncu_full.log 2>&1
echo ncu_full rc=$? >> $O/plain2.log

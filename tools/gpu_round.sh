#!/bin/bash
# GPU evidence run: gpu tests, smoke, default bench, C1-C4 configs, optional ncu.
# usage: tools/gpu_round.sh TAG [steps...]   steps: tests smoke bench ref configs refconfigs f3 f4 list solve probe
set -u
O=gpurun_out
T=${1:-x}; shift
STEPS=${*:-"tests smoke bench"}
make -s all >/dev/null 2>&1 || { echo build failed; exit 1; }
nproc > $O/host_$T.txt; lscpu >> $O/host_$T.txt 2>&1
for s in $STEPS; do
case $s in
probe) (find / -xdev -name SimplicialCholesky 2>/dev/null; find / -xdev -path '*Eigen/Dense' 2>/dev/null; echo done) > $O/eigen_probe_$T.txt ;;
tests) timeout 1800 python -m pytest tests -m gpu -q -p no:hypothesispytest > $O/pytest_$T.log 2>&1; echo rc=$? >> $O/pytest_$T.log ;;
smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$T.log 2>&1; echo rc=$? >> $O/smoke_$T.log ;;
bench) timeout 900 python bench.py > $O/bench_$T.log 2>&1; echo rc=$? >> $O/bench_$T.log ;;
ref) timeout 900 python bench.py --impl reference > $O/bench_ref_$T.log 2>&1; echo rc=$? >> $O/bench_ref_$T.log ;;
configs) for C in C1 C2 C3 C4; do timeout 900 python bench.py --config $C --steps 3 --warmup 3 > $O/bench_${C}_$T.log 2>&1; echo rc=$? >> $O/bench_${C}_$T.log; done ;;
refconfigs) for C in C1 C2 C3 C4; do timeout 900 python bench.py --config $C --impl reference --steps 3 --warmup 1 > $O/bench_ref_${C}_$T.log 2>&1; echo rc=$? >> $O/bench_ref_${C}_$T.log; done ;;
f3) timeout 600 python bench.py --config F3 --steps 3 --warmup 3 > $O/bench_f3_$T.log 2>&1; echo rc=$? >> $O/bench_f3_$T.log ;;
f4) timeout 600 python bench.py --config F4 --steps 20 --warmup 3 > $O/bench_f4_$T.log 2>&1; echo rc=$? >> $O/bench_f4_$T.log ;;
list) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 6100 -c 6100 --csv --log-file $O/launches_$T.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_list_$T.log 2>&1; echo rc=$? >> $O/ncu_list_$T.log ;;
solve) timeout 900 ncu --set full --clock-control none --import-source on -k regex:solve -s 40 -c 2 -o $O/prof_solve_$T python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_$T.log 2>&1; echo rc=$? >> $O/ncu_full_$T.log ;;
esac
done

#!/bin/bash
set -u
O=gpurun_out
T=${1:-x}
make -s all tools >/dev/null 2>&1 || { echo build failed; exit 1; }
{ build/solve_bench 32 200 20 32 1; build/solve_bench 32 200 20 64 1; } > $O/solve_$T.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:hypothesispytest > $O/pytest_$T.log 2>&1; echo rc=$? >> $O/pytest_$T.log
timeout 600 python bench.py --config F4 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_f4_$T.log 2>&1; echo rc=$? >> $O/bench_f4_$T.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$T.log 2>&1; echo rc=$? >> $O/bench_$T.log

#!/bin/bash
# iteration run: solve timing probes, full gpu test suite, C5 bench (no CPU leg)
set -u
O=gpurun_out
T=${1:-x}
make -s all tools >/dev/null 2>&1 || { echo build failed; exit 1; }
{
for W in 32 64; do
  for v in solve_bench solve_bench_nomma; do
    echo -n "$v: "; build/$v 32 200 20 $W 1
  done
done
echo -n "B=1: "; build/solve_bench 1 200 20 32 1
echo -n "B=1: "; build/solve_bench 1 200 20 64 1
} > $O/solve_$T.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:hypothesispytest > $O/pytest_$T.log 2>&1; echo rc=$? >> $O/pytest_$T.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$T.log 2>&1; echo rc=$? >> $O/bench_$T.log

#!/bin/bash
# standalone solve timing variants (tools/solve_bench.cu) + Cholesky phase probes
set -u
O=gpurun_out
T=${1:-x}
make -s tools >/dev/null 2>&1 || { echo build failed; exit 1; }
{
for W in 32; do
  for v in solve_bench solve_bench_nomma solve_bench_norhs solve_bench_noslab solve_bench_nomma_norhs solve_bench_nomma_noslab solve_bench_ns5 solve_bench_nomma_ns5; do
    echo -n "$v: "; build/$v 32 200 20 $W 1
  done
done
for c in 200 400; do build/chol_bench 1 $c 20; build/chol_bench 32 $c 10; done
} > $O/solve_exp_$T.log 2>&1

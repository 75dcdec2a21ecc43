#!/bin/bash
# Kernel probes: solve data-movement variants, Gram split-K sweep, ncu captures
# of the Gram / Cholesky / solve launches of one C5 step.
# usage: tools/gpu_probe.sh TAG [steps...]   steps: solve splits ncu
set -u
O=gpurun_out
T=${1:-p}; shift
STEPS=${*:-"solve splits ncu"}
make -s -j16 all tools >/dev/null 2>&1 || { echo build failed; exit 1; }
for s in $STEPS; do
case $s in
solve)
  for v in ${SOLVE_VARIANTS:-solve_bench solve_bench_halfslab solve_bench_noslab solve_bench_norhs solve_bench_nomma}; do
    echo "== $v" >> $O/probe_solve_$T.txt
    timeout 120 ./build/$v 32 200 20 32 1 >> $O/probe_solve_$T.txt 2>&1
    timeout 120 ./build/$v 64 200 20 32 1 >> $O/probe_solve_$T.txt 2>&1
  done ;;
splits)
  for k in 0 3 6 8; do
    if [ $k = 0 ]; then E=""; else E="SMG_GRAM_SPLITS=$k"; fi
    echo "== splits $k" >> $O/probe_splits_$T.txt
    env $E timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms_per_step'])" >> $O/probe_splits_$T.txt 2>&1
  done ;;
ncu)
  CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"gemm_pipe_kernel<1, 0, 4, 2>|gemm_pipe_kernel<0, 0, 4, 2>|cholx_kernel|solve_kernel<32, 16>|chol_kernel" \
    -s 400 -c 6 -o $O/prof_probe_$T $CMD > $O/ncu_probe_$T.log 2>&1; echo rc=$? >> $O/ncu_probe_$T.log ;;
ncuproj)
  CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"recon_mma|partial_kernel|rank_partial|chunk_reduce|gemm_pipe_kernel<false, false, 4, 2" -s 300 -c 10 -o $O/prof_proj_$T $CMD > $O/ncu_proj_$T.log 2>&1; echo rc=$? >> $O/ncu_proj_$T.log ;;
ab)
  # back-to-back A/B of environment variants (AB_VARIANTS="name=ENV ..."), twice each
  for rep in 1 2; do
    for v in ${AB_VARIANTS:-base=X}; do
      name=${v%%=*}; envs=${v#*=}; envs=${envs//,/ }
      r=$(env $envs timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), d['stages_ms_per_step'])")
      echo "$name rep$rep $r" >> $O/probe_ab_$T.txt
    done
  done ;;
debug)
  SMG_DEBUG=1 timeout 600 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/debug_$T.log 2>&1 ;;
tests)
  timeout 1800 python -m pytest tests -m gpu -q -x -p no:hypothesispytest > $O/pytest_$T.log 2>&1; echo rc=$? >> $O/pytest_$T.log ;;
bench)
  timeout 900 python bench.py > $O/bench_$T.log 2>&1; echo rc=$? >> $O/bench_$T.log ;;
esac
done

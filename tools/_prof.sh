set -u
O=gpurun_out
make -s all >/dev/null 2>&1 || exit 1
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_pipe_kernel -s 400 -c 4 -o $O/prof_gemm_r02g $CMD > $O/ncu_gemm_r02g.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 100 -c 1 -o $O/prof_solve_r02g $CMD > $O/ncu_solve_r02g.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chol_kernel -s 100 -c 2 -o $O/prof_chol_r02g $CMD > $O/ncu_chol_r02g.log 2>&1

set -u
O=gpurun_out
make -s all >/dev/null 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:hypothesispytest > $O/pytest_r02f.log 2>&1; echo rc=$? >> $O/pytest_r02f.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_r02f.log 2>&1
SMG_ORTH_SKIP_TOL=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_r02f_noskip.log 2>&1
for m in 8 16 32; do timeout 600 python bench.py --meshes $m --steps 5 --warmup 3 --no-cpu-baseline > $O/sweep2_m$m.log 2>&1; done
for gsz in 4 8; do SMG_GROUPS=$gsz timeout 600 python bench.py --meshes 8 --steps 5 --warmup 3 --no-cpu-baseline > $O/sweep2_m8_g$gsz.log 2>&1; done

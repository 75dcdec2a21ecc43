set -u
O=gpurun_out
make -s all >/dev/null 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:hypothesispytest > $O/pytest_trsm.log 2>&1; echo rc=$? >> $O/pytest_trsm.log
timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > $O/trsm_c4.log 2>&1
timeout 600 python bench.py --meshes 8 --steps 5 --warmup 3 --no-cpu-baseline > $O/trsm_m8.log 2>&1
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > $O/trsm_c2.log 2>&1

set -u
O=gpurun_out
make -s all >/dev/null 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:hypothesispytest > $O/pytest_r02k.log 2>&1; echo rc=$? >> $O/pytest_r02k.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/w_c5.log 2>&1
timeout 600 python bench.py --meshes 8 --steps 5 --warmup 3 --no-cpu-baseline > $O/w_m8.log 2>&1
for C in C1 C2 C3 C4; do timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline > $O/w_$C.log 2>&1; done

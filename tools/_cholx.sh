set -u
O=gpurun_out
make -s all >/dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_chain.py -q -x -p no:hypothesispytest > $O/pytest_cholx.log 2>&1; echo rc=$? >> $O/pytest_cholx.log

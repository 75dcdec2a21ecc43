#!/bin/bash
# tests + default bench + 8-mesh bench (per-rank load at N=8)
set -u
O=gpurun_out
TAG=${1:-x}
make -s >/dev/null 2>&1 || { echo build failed; exit 1; }
python -m pytest tests -m gpu -x -q -p no:hypothesispytest > $O/pytest_$TAG.log 2>&1; echo rc=$? >> $O/pytest_$TAG.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$TAG.log 2>&1; echo rc=$? >> $O/bench_$TAG.log
python bench.py --meshes 8 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_m8_$TAG.log 2>&1; echo rc=$? >> $O/bench_m8_$TAG.log

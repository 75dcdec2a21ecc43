#!/bin/bash
# tests (all gpu), smoke, configs C1-C4 throughput, F3 launch-free
set -u
O=gpurun_out
T=${1:-r01e}
make -s >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:hypothesispytest > $O/pytest_$T.log 2>&1; echo rc=$? >> $O/pytest_$T.log
timeout 900 python tools/bench_configs.py > $O/configs_$T.log 2>&1; echo rc=$? >> $O/configs_$T.log

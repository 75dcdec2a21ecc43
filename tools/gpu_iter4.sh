#!/bin/bash
set -u
O=gpurun_out
T=${1:-x}
make -s all >/dev/null 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x -p no:hypothesispytest > $O/pytest_$T.log 2>&1; echo rc=$? >> $O/pytest_$T.log
timeout 900 python tools/bench_configs.py > $O/configs_$T.log 2>&1; echo rc=$? >> $O/configs_$T.log

set -u
O=gpurun_out
make -s all >/dev/null 2>&1 || exit 1
SMG_DOI_NOGRAPH=1 timeout 600 python bench.py --config C4 --steps 2 --warmup 3 --no-cpu-baseline > $O/c4ng.log 2>&1
SMG_DOI_NOGRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 4000 -c 4000 --csv --log-file $O/launches_c4ng.csv python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_c4ng.log 2>&1

set -u
O=gpurun_out
make -s all >/dev/null 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 3000 --csv --log-file $O/launches_c4_r02h.csv python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_c4_r02h.log 2>&1; echo rc=$? >> $O/ncu_c4_r02h.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 2000 --csv --log-file $O/launches_c2_r02h.csv python bench.py --config C2 --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_c2_r02h.log 2>&1; echo rc=$? >> $O/ncu_c2_r02h.log

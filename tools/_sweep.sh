set -u
O=gpurun_out
make -s all >/dev/null 2>&1 || exit 1
for m in 8 16 32; do timeout 600 python bench.py --meshes $m --steps 5 --warmup 3 --no-cpu-baseline > $O/sweep_m$m.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 6000 --csv --log-file $O/launches_r02e.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_list_r02e.log 2>&1; echo rc=$? >> $O/ncu_list_r02e.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 1500 --csv --log-file $O/launches_m8_r02e.csv python bench.py --meshes 8 --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_list_m8_r02e.log 2>&1

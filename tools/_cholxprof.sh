set -u
O=gpurun_out
make -s all >/dev/null 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cholx -s 20 -c 1 -o $O/prof_cholx_c2 python bench.py --config C2 --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_cholx_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cholx -s 20 -c 1 -o $O/prof_cholx_c5 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_cholx_c5.log 2>&1

set -u
O=gpurun_out
make -s all >/dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -p no:hypothesispytest -k "chain or config or primitives or frames or codec" > $O/pytest_rec.log 2>&1; echo rc=$? >> $O/pytest_rec.log
for v in 2 3 6; do SMG_RECON_CPS=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/rec_$v.log 2>&1; done
SMG_RECON_OLD=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/rec_old.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:recon -s 20 -c 6 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_rec.csv 2>&1

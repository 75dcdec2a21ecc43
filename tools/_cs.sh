set -u
O=gpurun_out
make -s all >/dev/null 2>&1 || exit 1
for cs in 32 16; do SMG_SOLVE_CS=$cs timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/cs_c5_$cs.log 2>&1; done
for cs in 32 16 8; do SMG_SOLVE_CS=$cs timeout 600 python bench.py --meshes 8 --steps 5 --warmup 3 --no-cpu-baseline > $O/cs_m8_$cs.log 2>&1; done
for g in geometric natural; do SMG_ORDERING=$g timeout 600 python bench.py --meshes 8 --steps 5 --warmup 3 --no-cpu-baseline > $O/ord_m8_$g.log 2>&1; done
for cs in 16 8; do SMG_SOLVE_CS=$cs timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > $O/cs_c4_$cs.log 2>&1; done

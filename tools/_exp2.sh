set -u
O=gpurun_out
make -s all >/dev/null 2>&1 || exit 1
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > $O/x_c2_$tag.log 2>&1; env "$@" timeout 600 python bench.py --meshes 8 --steps 5 --warmup 3 --no-cpu-baseline > $O/x_m8_$tag.log 2>&1; env "$@" timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > $O/x_c4_$tag.log 2>&1; }
run base X=1
run minp7 SMG_CHOL_CLUSTER_MINP=4
run minp7b8 SMG_CHOL_CLUSTER_MINP=4 SMG_CHOL_CLUSTER_MAXB=8

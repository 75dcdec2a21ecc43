cd $GRAFT_REPO_ROOT
for args in "1 100 20 1 1" "1 100 20 4 1" "1 200 20 1 0" "1 200 20 2 1" "1 200 20 8 1" "32 200 10 2 0" "1 400 10 4 1" "1 400 10 8 1" "1 400 10 8 0"; do timeout 60 ./build/cholx_bench $args; done > gpurun_out/cxb.log 2>&1

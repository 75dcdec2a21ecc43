#!/bin/bash
O=gpurun_out
for cfg in "16 3" "32 2" "32 3" "24 3"; do
  set -- $cfg
  touch paper_1810_02719_b200/csrc/gemm.cu
  make -s -j16 all EXTRA="-DSMG_GEMM_BKP=$1 -DSMG_GEMM_PNS=$2" >/dev/null 2>&1 || { echo "build fail $cfg" >> $O/bkp.log; continue; }
  echo -n "BKP=$1 PNS=$2: " >> $O/bkp.log
  python bench.py --steps 2 --warmup 2 --no-cpu-baseline 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k: d['stages_ms_per_step'][k] for k in ('gram','trmm','orthonormalize','first_basis')})" >> $O/bkp.log 2>&1
done

#!/bin/bash
# 4-per-SM backprojector and 24-angle small-batch forward projector A/B on rank shards
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for wr in "8 3" "8 0" "4 1" "1 0"; do
  set -- $wr
  for envs in "LT_BP_MINB4=0 LT_FP_ONE=1" "LT_BP_MINB4=0" "LT_BP_MINB4=1" "LT_FP_ONE=-1"; do
    echo "w$1 r$2 [$envs] $(env $envs KB_WORLD=$1 KB_RANK=$2 KB_NITER=12 python tools/kernel_bench.py C4 2>&1 | tail -1)"
  done
  echo "w$1 r$2 [default] $(SH_WORLD=$1 SH_RANK=$2 SH_NITER=50 python tools/shard_time.py C4 2>&1 | tail -1)"
  echo "w$1 r$2 [old]     $(LT_BP_MINB4=0 LT_FP_ONE=1 SH_WORLD=$1 SH_RANK=$2 SH_NITER=50 python tools/shard_time.py C4 2>&1 | tail -1)"
done

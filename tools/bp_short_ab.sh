#!/bin/bash
# 64x32 ROI-backprojection sub-tiles (LT_BP_SHORT: unset = rule, 0 off, 1 force) on rank shards and C3
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for wr in "8 3" "8 0" "4 1" "2 0"; do
  set -- $wr
  for v in 0 1; do
    echo "w$1 r$2 [SHORT=$v] $(LT_BP_SHORT=$v KB_WORLD=$1 KB_RANK=$2 KB_NITER=12 TAG=s$v python tools/kernel_bench.py C4 2>&1 | tail -1)"
  done
  python -c "
import torch; a=torch.load('/tmp/lt_ab/cores_s0.pt'); b=torch.load('/tmp/lt_ab/cores_s1.pt'); print('  rel diff', float((a-b).norm()/a.norm()))"
  echo "w$1 r$2 [rule] $(SH_WORLD=$1 SH_RANK=$2 SH_NITER=50 python tools/shard_time.py C4 2>&1 | tail -1)"
  echo "w$1 r$2 [off]  $(LT_BP_SHORT=0 SH_WORLD=$1 SH_RANK=$2 SH_NITER=50 python tools/shard_time.py C4 2>&1 | tail -1)"
done
for c in C3 C5; do for v in 0 1; do echo "$c [SHORT=$v] $(LT_BP_SHORT=$v KB_NITER=8 python tools/kernel_bench.py $c 2>&1 | tail -1)"; done; done

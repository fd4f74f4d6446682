#!/bin/bash
# Two-group pipelining with one shared side-stream x_s (LT_SPLIT=2, LT_SPLIT_B = second group's size)
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
export SH_NITER=${SH_NITER:-50}
for wr in "8 3" "8 0" "4 1"; do
  set -- $wr
  echo "w$1 r$2 base        $(SH_WORLD=$1 SH_RANK=$2 python tools/shard_time.py C4 2>&1 | tail -1)"
  for b in 1 2 4; do
    echo "w$1 r$2 B=$b         $(LT_SPLIT=2 LT_SPLIT_B=$b SH_WORLD=$1 SH_RANK=$2 python tools/shard_time.py C4 2>&1 | tail -1)"
  done
  echo "w$1 r$2 B=2 oldxs    $(LT_SPLIT_XS=0 LT_SPLIT=2 LT_SPLIT_B=2 SH_WORLD=$1 SH_RANK=$2 python tools/shard_time.py C4 2>&1 | tail -1)"
done
echo "w1 base   $(python tools/shard_time.py C4 2>&1 | tail -1)"
for b in 1 16 31; do echo "w1 B=$b   $(LT_SPLIT=2 LT_SPLIT_B=$b python tools/shard_time.py C4 2>&1 | tail -1)"; done

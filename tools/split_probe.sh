#!/bin/bash
# Two-group pipelining A/B (LT_SPLIT=2, LT_SPLIT_B = size of the second group) on rank shards
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
export SH_NITER=${SH_NITER:-50}
for r in 2 5; do
  echo "base      $(SH_WORLD=8 SH_RANK=$r python tools/shard_time.py C4 2>&1 | tail -1)"
  for b in 0 2 4 6; do
    echo "split B=$b $(LT_SPLIT=2 LT_SPLIT_B=$b SH_WORLD=8 SH_RANK=$r python tools/shard_time.py C4 2>&1 | tail -1)"
    echo "split B=$b noprio $(LT_PRIO=0 LT_SPLIT=2 LT_SPLIT_B=$b SH_WORLD=8 SH_RANK=$r python tools/shard_time.py C4 2>&1 | tail -1)"
  done
done
echo "w1 base   $(python tools/shard_time.py C4 2>&1 | tail -1)"
for b in 1 16; do
echo "w1 B=$b   $(LT_SPLIT=2 LT_SPLIT_B=$b python tools/shard_time.py C4 2>&1 | tail -1)"
done

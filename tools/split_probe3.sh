#!/bin/bash
# One-GPU C4: two-group pipelining with a shared side-stream x_s, second-group sizes
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
export SH_NITER=200 SH_REPS=3
echo "base  $(python tools/shard_time.py C4 2>&1 | tail -1)"
for b in 1 16 31 46 61 128; do echo "B=$b  $(LT_SPLIT=2 LT_SPLIT_B=$b python tools/shard_time.py C4 2>&1 | tail -1)"; done
echo "base  $(python tools/shard_time.py C4 2>&1 | tail -1)"
echo "B=31 noprio $(LT_PRIO=0 LT_SPLIT=2 LT_SPLIT_B=31 python tools/shard_time.py C4 2>&1 | tail -1)"

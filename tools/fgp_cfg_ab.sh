#!/bin/bash
# FGP launch-shape A/B (LT_FGP2_CFG) at world 1 and a world-8 shard of C4
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for cfg in "" 2x16b 2x8b 4x8; do
  echo "[$cfg] w1 $(LT_FGP2_CFG=$cfg KB_NITER=10 python tools/kernel_bench.py C4 2>&1 | tail -1)"
  echo "[$cfg] w8 $(LT_FGP2_CFG=$cfg KB_WORLD=8 KB_RANK=3 KB_NITER=20 python tools/kernel_bench.py C4 2>&1 | tail -1)"
done

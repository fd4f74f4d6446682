#!/bin/bash
# Partition cost weight A/B (LT_PART_FGPW) on the projected 8-GPU C4 step
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for w in 2 4 1 0; do
  echo "FGPW=$w"; LT_PART_FGPW=$w python tools/rank_scaling_detail.py C4 8 2>&1 | tail -9
done

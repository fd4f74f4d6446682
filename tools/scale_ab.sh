#!/bin/bash
# strong-scaling projection A/B (tools/rank_scaling.py) under environment variants
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in "" "LT_SPLIT=2" "LT_SPLIT=2 LT_PRIO=0"; do
  echo "== [$v]"
  env $v python tools/rank_scaling.py C4 ${WORLDS:-8} 2>&1 | tail -2
done

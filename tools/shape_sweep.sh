#!/bin/bash
# Launch-shape rule check across the small workloads: bench.py value under each forcing switch vs the rules
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
val() { env "$@" python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"])'; }
for CFG in C1 C2 C3 L1 T1 P1; do
  line="$CFG rule=$(val LT_X=1)"
  for v in "LT_BP_SUB=32" "LT_BP_SUB=64" "LT_GRAPH=0" "LT_GRAPH=1" "LT_FP_ONE=0" "LT_FP_ONE=1" "LT_FGP2_CFG=4x8" "LT_FGP2_CFG=2x8" "LT_BP_TALL=0"; do
    line="$line | $v=$(val $v)"
  done
  echo "$line"
done

#!/bin/bash
# A/B of the forward-projector zero margins on small tiles (C1 40^2, C2 / L1 128^2) and C4
bash tools/build_variant.sh xpad0 -DFP_XPAD=0
for c in C1 C2 L1 C4; do KB_NITER=20 bash tools/ab.sh $c "" "LT_SO=/tmp/lt_ab/xpad0.so"; done
for c in C1 L1 C2; do
  echo "$c new $(python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"])')"
  echo "$c old $(LT_SO=/tmp/lt_ab/xpad0.so python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"])')"
done

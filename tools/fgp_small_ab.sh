#!/bin/bash
# FGP launch shape on small batches: 16-row CTAs (2x8) vs 32-row CTAs (4x8) vs the rule
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for c in C2 L1 C3 T1 P1; do
  for cfg in "" 2x8 4x8; do
    echo "$c [$cfg] $(LT_FGP2_CFG=$cfg KB_NITER=12 python tools/kernel_bench.py $c 2>&1 | tail -1)"
  done
done

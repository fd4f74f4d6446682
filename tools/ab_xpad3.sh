#!/bin/bash
# A/B of the forward-projector zero margins (two-angles-per-warp kernels only) across configs
bash tools/build_variant.sh xpad0 -DFP_XPAD=0
for c in L1 C3 C4 T1; do KB_NITER=20 bash tools/ab.sh $c "" "LT_SO=/tmp/lt_ab/xpad0.so"; done
KB_NITER=10 bash tools/ab.sh C5 "" "LT_SO=/tmp/lt_ab/xpad0.so"

#!/bin/bash
# A/B: zero margins on the staged forward-projector lines (FP_XPAD=16, default) vs none (-DFP_XPAD=0)
bash tools/build_variant.sh xpad0 -DFP_XPAD=0
KB_NITER=20 bash tools/ab.sh C4 "" "LT_SO=/tmp/lt_ab/xpad0.so"
KB_NITER=10 bash tools/ab.sh C5 "" "LT_SO=/tmp/lt_ab/xpad0.so"
KB_NITER=20 bash tools/ab.sh C3 "" "LT_SO=/tmp/lt_ab/xpad0.so"
KB_NITER=20 bash tools/ab.sh P1 "" "LT_SO=/tmp/lt_ab/xpad0.so"

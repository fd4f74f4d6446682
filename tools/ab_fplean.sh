#!/bin/bash
# A/B: FP_LEAN (default) vs the round-2 projector setup (-DFP_LEAN=0)
bash tools/build_variant.sh fp_old -DFP_LEAN=0
KB_NITER=20 bash tools/ab.sh C4 "" "LT_SO=/tmp/lt_ab/fp_old.so"
KB_NITER=10 bash tools/ab.sh C5 "" "LT_SO=/tmp/lt_ab/fp_old.so"
KB_NITER=20 bash tools/ab.sh C3 "" "LT_SO=/tmp/lt_ab/fp_old.so"

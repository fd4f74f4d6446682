#!/bin/bash
# A/B: 32-line projector bands (-DFP_BLN=32) vs the default 16
bash tools/build_variant.sh bl32 -DFP_BLN=32
KB_NITER=20 bash tools/ab.sh C4 "" "LT_SO=/tmp/lt_ab/bl32.so"
KB_NITER=10 bash tools/ab.sh C5 "" "LT_SO=/tmp/lt_ab/bl32.so"

#!/bin/bash
# A/B of the CP = 4 FGP address keeping: default (none) vs the mbarrier base only (1) vs all (2)
bash tools/build_variant.sh keep1 -DFGP_KEEP4=1
bash tools/build_variant.sh keep2 -DFGP_KEEP4=2
for i in 1 2; do KB_NITER=30 bash tools/ab.sh C4 "" "LT_SO=/tmp/lt_ab/keep1.so" "LT_SO=/tmp/lt_ab/keep2.so"; done

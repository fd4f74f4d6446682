#!/bin/bash
bash tools/build_variant.sh fgp_old -DFGP_OPAQUE=0
for c in C4 C4 C3; do KB_NITER=30 bash tools/ab.sh $c "" "LT_SO=/tmp/lt_ab/fgp_old.so" "" "LT_SO=/tmp/lt_ab/fgp_old.so"; done

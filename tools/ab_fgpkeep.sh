#!/bin/bash
# A/B: FGP loop-invariant shared addresses kept in registers (default) vs rematerialised (-DFGP_OPAQUE=0)
bash tools/build_variant.sh fgp_old -DFGP_OPAQUE=0
for c in C4 C3 L1 P1; do KB_NITER=20 bash tools/ab.sh $c "" "LT_SO=/tmp/lt_ab/fgp_old.so"; done

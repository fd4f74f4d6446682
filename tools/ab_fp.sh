#!/bin/bash
# FP staging / double-buffer A/B (round 2)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/build_variant.sh v_st0 -DFP_STAGE64=0
KB_NITER=20 bash tools/ab.sh C4 "" "LT_FP_NBUF=1" "LT_SO=gpurun_out/v_st0.so" "LT_SO=gpurun_out/v_st0.so LT_FP_NBUF=1"

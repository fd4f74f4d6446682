#!/bin/bash
# Forward-projector launch shape for small batches: 8-angle CTAs (LT_FP_ONE=1) vs 24/16-angle CTAs (LT_FP_ONE=0) vs the rule
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
run() { # cfg world rank
  for v in "" 0 1; do
    echo "$1 w$2 r$3 [FP_ONE=$v] $(LT_FP_ONE=$v KB_WORLD=$2 KB_RANK=$3 KB_NITER=12 python tools/kernel_bench.py $1 2>&1 | tail -1)"
  done
}
run C4 4 1; run C4 8 3; run C4 8 0; run C3 1 0; run C2 1 0; run L1 1 0; run C5 8 3; run C5 16 5

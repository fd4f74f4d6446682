#!/bin/bash
# Per-kernel timing of every rank shard of C4 at world = 8 (and world = 1) on one B200.
set -u
for r in 0 1 2 3 4 5 6 7; do
  echo "w8 r$r $(KB_WORLD=8 KB_RANK=$r KB_NITER=20 python tools/kernel_bench.py C4 2>&1 | tail -1)"
done
echo "w1 $(KB_NITER=20 python tools/kernel_bench.py C4 2>&1 | tail -1)"

#!/bin/bash
# A/B of kernel variants selected by environment switches (each in its own process):
#   bash tools/ab.sh <config> "<ENV=..>" "<ENV=..>" ...   ("" = defaults)
# prints per-class average launch times of tools/kernel_bench.py and the max |diff| of the cores vs the first variant
cfg=$1; shift
mkdir -p gpurun_out
i=0
for v in "$@"; do
  env $v TAG=ab$i KB_NITER=${KB_NITER:-20} python tools/kernel_bench.py $cfg 2>&1 | tail -1 | sed "s|^|[$v] |"
  i=$((i+1))
done
python - "$i" <<'PY'
import sys, torch
n = int(sys.argv[1])
a = torch.load("/tmp/lt_ab/cores_ab0.pt")
for k in range(1, n):
    b = torch.load(f"/tmp/lt_ab/cores_ab{k}.pt")
    print(f"variant {k}: max|diff| vs 0 = {float((a - b).abs().max()):.3e}, rel = {float((a - b).norm() / a.norm()):.3e}")
PY

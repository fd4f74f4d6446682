#!/bin/bash
# Launch-shape A/B on a C4 rank shard at world = 8 (kernel classes via lt_timing and solve time)
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
export SH_NITER=${SH_NITER:-50} SH_WORLD=8 SH_RANK=${SH_RANK:-3}
for envs in "" "LT_FP_ONE=0" "LT_BP_SUB=64" "LT_FP_ONE=0 LT_BP_SUB=64" "LT_BP_TALL=0 LT_BP_SUB=64" "LT_FGP2_CFG=2x8" "LT_GRAPH=1" "LT_XS_OVERLAP=0"; do
  echo "[$envs] $(env $envs python tools/shard_time.py C4 2>&1 | tail -1)"
  echo "[$envs] $(env $envs KB_WORLD=8 KB_RANK=$SH_RANK KB_NITER=20 python tools/kernel_bench.py C4 2>&1 | tail -1)"
done

#!/bin/bash
# Profile capture for profiles/<round>/ (run on the GPU box via gpurun):
#   1. launch list of one bench step (ncu --metrics gpu__time_duration.sum, clocks free)
#   2. ncu --set full of one launch of each hot kernel (k_fgp2, k_fp_roi2, k_bp ROI / global)
# Output in gpurun_out/prof_<tag>*; summarise with tools/launch_summary.py, tools/ncu_summary.py.
set -u
TAG=${1:-v}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_${TAG}_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof_${TAG}_launch.log 2>&1
python tools/launch_summary.py gpurun_out/prof_${TAG}_launches.csv > gpurun_out/prof_${TAG}_launch_summary.txt
ncu --set full --import-source on --clock-control none -k regex:"k_fgp2|k_fp_roi2|k_bp" --launch-skip 12 -c 4 \
    -o gpurun_out/prof_${TAG}_full python tools/kernel_bench.py > gpurun_out/prof_${TAG}_full.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_${TAG}_full.ncu-rep > gpurun_out/prof_${TAG}_full_summary.txt
ncu -i gpurun_out/prof_${TAG}_full.ncu-rep --page details --csv > gpurun_out/prof_${TAG}_full_details.csv 2>/dev/null
cat gpurun_out/prof_${TAG}_launch_summary.txt gpurun_out/prof_${TAG}_full_summary.txt

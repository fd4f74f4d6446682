#!/bin/bash
# Profile capture for profiles/<round>/ (run on the GPU box via gpurun):
#   1. launch list of one bench step (ncu --metrics gpu__time_duration.sum, clocks free)
#   2. ncu --set full of one launch of each hot kernel of the C4 solve
#      (k_fgp2, the ROI k_fp_roi2, the ROI k_bp<1,3>, the global x_s k_bp<1,1>)
# Output in gpurun_out/prof_<tag>*; summarised with tools/launch_summary.py, tools/ncu_summary.py.
set -u
TAG=${1:-v}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_${TAG}_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof_${TAG}_launch.log 2>&1
python tools/launch_summary.py gpurun_out/prof_${TAG}_launches.csv > gpurun_out/prof_${TAG}_launch_summary.txt
# kernel_bench: bank (6 tiled global FPs) + disc W.D (1) precede the solves' ROI FPs
full() {  # name filter, launch skip, output suffix
    ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k "regex:$1" \
        --launch-skip "$2" -c 1 -o "gpurun_out/prof_${TAG}_$3" python tools/kernel_bench.py > /dev/null 2>&1
    python tools/ncu_summary.py "gpurun_out/prof_${TAG}_$3.ncu-rep"
    ncu -i "gpurun_out/prof_${TAG}_$3.ncu-rep" --page details --csv > "gpurun_out/prof_${TAG}_$3_details.csv" 2>/dev/null
}
{
    full "k_fgp2" 0 fgp
    full "k_fp_roi2" 8 fp
    full "k_bpILi1ELi3E" 0 bp
    full "k_bpILi1ELi1E" 0 xs
} > gpurun_out/prof_${TAG}_full_summary.txt
cat gpurun_out/prof_${TAG}_launch_summary.txt gpurun_out/prof_${TAG}_full_summary.txt

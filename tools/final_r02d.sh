#!/bin/bash
# Round-2 (session 2) evidence refresh at HEAD: ncu captures (prof_r02d), SASS stall tables, then the end-of-round runs
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02d_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1500 bash tools/profile_round.sh r02d > gpurun_out/r02d_profile.log 2>&1; echo "profile rc=$?"
for k in fgp fp bp; do python tools/ncu_sass_stalls.py gpurun_out/prof_r02d_$k.ncu-rep > gpurun_out/prof_r02d_${k}_sass_stalls.txt 2>&1; done
bash tools/final_runs.sh

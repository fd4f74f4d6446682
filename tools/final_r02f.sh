#!/bin/bash
# Round-2 (session 2) evidence refresh at HEAD: ncu captures (prof_r02f), SASS stall tables, then the end-of-round runs
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02f_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1500 bash tools/profile_round.sh r02f > gpurun_out/r02f_profile.log 2>&1; echo "profile rc=$?"
for k in fgp fp bp; do python tools/ncu_sass_stalls.py gpurun_out/prof_r02f_$k.ncu-rep > gpurun_out/prof_r02f_${k}_sass_stalls.txt 2>&1; done
bash tools/final_runs.sh
# random-geometry parity sweep at the final build (new launch shapes included)
LT_FUZZ_SEEDS=600 LT_FUZZ_WIDE=120 timeout 1800 python -m pytest tests/test_fuzz_parity.py -m gpu -q > gpurun_out/final_fuzz600.txt 2>&1; echo "fuzz rc=$?"; tail -1 gpurun_out/final_fuzz600.txt

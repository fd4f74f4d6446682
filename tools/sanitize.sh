#!/bin/bash
# One compute-sanitizer tool over every case of tools/sanitize_cases.py (one tool per gpurun call).
# Usage: bash tools/sanitize.sh memcheck|racecheck|synccheck [cases...]
tool=$1; shift
cases=${*:-C1 C2 T1 P}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in $cases; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --kernel-name kns=_ZN2lt \
    --print-limit 50 python tools/sanitize_cases.py $c > gpurun_out/san_${tool}_${c}.txt 2>&1
  echo "$tool $c rc=$? : $(tail -1 gpurun_out/san_${tool}_${c}.txt)"
done

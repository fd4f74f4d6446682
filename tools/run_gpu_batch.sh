#!/bin/bash
# Round-2 GPU batch: peaks microbenchmark, new GPU tests, default bench.
# Usage (from the repo root, through gpurun): bash tools/run_gpu_batch.sh <tag> [pytest -k expr]
set -u
tag=${1:-a}
kexpr=${2:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
nproc > gpurun_out/${tag}_host.txt; lscpu >> gpurun_out/${tag}_host.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/${tag}_build.log; exit 1; }
[ -x tools/peaks_micro ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/peaks_micro tools/peaks_micro.cu
timeout 120 tools/peaks_micro > gpurun_out/${tag}_peaks_micro.json 2>&1; echo "peaks rc=$?"
if [ -n "$kexpr" ]; then
  LT_PARITY_REPORT=gpurun_out/${tag}_parity.jsonl timeout 1500 python -m pytest tests -m gpu -x -q -k "$kexpr" > gpurun_out/${tag}_pytest.log 2>&1
  echo "pytest rc=$?"; tail -5 gpurun_out/${tag}_pytest.log
fi
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"; tail -c 600 gpurun_out/${tag}_bench.json

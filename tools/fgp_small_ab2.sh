#!/bin/bash
# FGP shape rule for narrow tiles (CP <= 2): kernel times and bench lines
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for c in C2 L1; do echo "$c $(KB_NITER=12 python tools/kernel_bench.py $c 2>&1 | tail -1)"; done
for c in L1 C2; do echo "$c bench $(python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["e2e"]["value"])')"; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fuzz_parity.py -m gpu -x -q 2>&1 | tail -2

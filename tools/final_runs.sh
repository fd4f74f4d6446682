#!/bin/bash
# End-of-round runs on one B200 (outputs in gpurun_out/final_*; summaries copied to profiles/r02 by hand)
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final_build.log 2>&1 || { echo BUILD FAILED; exit 1; }
LT_PARITY_REPORT=gpurun_out/final_parity.jsonl timeout 2400 python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/final_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/final_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench_C4.json 2> gpurun_out/final_bench_C4.err; echo "bench C4 rc=$?"
for c in C1 C2 C3 C5 T1 L1 P1; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/final_bench_$c.json 2> gpurun_out/final_bench_$c.err; echo "bench $c rc=$?"
done
timeout 900 python bench.py --prior haar --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/final_bench_C4_haar.json 2>/dev/null; echo "haar rc=$?"
timeout 900 python bench.py --config C5 --prior exterior --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/final_bench_C5_exterior.json 2>/dev/null; echo "exterior rc=$?"
timeout 900 python bench.py --xs-exact --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/final_bench_C4_xsexact.json 2>/dev/null; echo "xs-exact rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_bench_ref.json 2>/dev/null; echo "ref rc=$?"
timeout 900 python tools/rank_scaling.py C4 > gpurun_out/final_rank_scaling.txt 2>&1; echo "scaling rc=$?"
timeout 900 python tools/rank_scaling.py C5 1,8 > gpurun_out/final_rank_scaling_C5.txt 2>&1; echo "scaling C5 rc=$?"
for c in C4 C2 C3 L1 P1 T1; do echo "$c $(KB_NITER=20 python tools/kernel_bench.py $c 2>&1 | tail -1)"; done > gpurun_out/final_kernel_bench.txt
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/final_bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        rf = d.get("roofline") or {}
        print(f"{f[18:]:32s} value={d.get('value')} e2e={(d.get('e2e') or {}).get('value')} frac={rf.get('frac')} ({rf.get('kernel')})")
    except Exception as e:
        print(f, "unreadable", e)
PY

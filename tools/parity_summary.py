"""Markdown table of a LT_PARITY_REPORT JSON-lines file (tests/test_gpu_full_iterations.py):
python tools/parity_summary.py profiles/r02/parity_full_iterations.jsonl"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
print("| Config | What | k / n | Max relL2 | Tolerance |")
print("|---|---|---|---|---|")
for r in rows:
    val = r.get("max_relL2", r.get("relL2", r.get("relerr")))
    kn = r.get("k", r.get("n_iter", ""))
    if r.get("n_fgp"):
        kn = f"{kn} x {r['n_fgp']}"
    print(f"| {r['config']} | {r['what']} | {kn} | {val:.2e} | {r['tol']:g} |")

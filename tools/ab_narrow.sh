python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python -m pytest tests -m gpu -x -q -k "fgp or tv or C1 or C2 or C3 or wide or fuzz or sweep or lambda" 2>&1 | tail -2
for c in C2 C3 L1; do
  for v in "" "LT_FGP_NARROW=0"; do echo "[$c $v]"; env $v KB_NITER=20 python tools/kernel_bench.py $c 2>&1 | tail -1; done
done
for c in C1 C2 C3 L1; do for v in "" "LT_FGP_NARROW=0"; do echo "[$c $v] $(env $v timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["rooflines"].get("fgp",{}).get("frac"))')"; done; done

python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python -m pytest tests/test_gpu_wide_tiles.py -x -q 2>&1 | tail -15
python -m pytest tests -m gpu -x -q -k "fgp or tv or C2 or guard or boundary" 2>&1 | tail -3
KB_NITER=20 bash tools/ab.sh C4 ""
timeout 300 python bench.py --config P1 --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-600

python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/build_variant.sh v_dyn -DFP_DYN=1
KB_NITER=20 bash tools/ab.sh C4 "" "LT_SO=/tmp/lt_ab/v_dyn.so"
for w in 8; do KB_WORLD=$w KB_NITER=20 python tools/kernel_bench.py C4 | tail -1; LT_SO=/tmp/lt_ab/v_dyn.so KB_WORLD=$w KB_NITER=20 python tools/kernel_bench.py C4 | tail -1; done
KB_NITER=20 python tools/kernel_bench.py C5 | tail -1; LT_SO=/tmp/lt_ab/v_dyn.so KB_NITER=20 python tools/kernel_bench.py C5 | tail -1

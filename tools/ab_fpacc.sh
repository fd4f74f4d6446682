python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/build_variant.sh v_acc1 -DFP_ACC2=0
KB_NITER=20 bash tools/ab.sh C4 "" "LT_SO=/tmp/lt_ab/v_acc1.so"

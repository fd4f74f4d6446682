python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/build_variant.sh v_pipe -DFP_PIPE=1
bash tools/build_variant.sh v_lea -DFP_LEA=1
KB_NITER=20 bash tools/ab.sh C4 "" "LT_SO=/tmp/lt_ab/v_pipe.so" "LT_SO=/tmp/lt_ab/v_lea.so" 2>&1 | grep -v "instantiation\|detected\|^ *^\|^$\|warning"

python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
KB_NITER=20 bash tools/ab.sh C4 "" "LT_FGP_PERSIST=0"
python -m pytest tests -m gpu -x -q -k "fgp or tv or lambda or sweep or haar or C2" 2>&1 | tail -3

#!/bin/bash
# Build the library with extra compile-time switches into /tmp/lt_ab/<name>.so (A/B only):
#   bash tools/build_variant.sh <name> -DFOO=1 ...   then  LT_SO=/tmp/lt_ab/<name>.so python ...
name=$1; shift
mkdir -p /tmp/lt_ab
/usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared \
  "$@" -I include -o /tmp/lt_ab/$name.so paper_1604_02292_b200/csrc/loctomo.cu -lcufft -Xlinker -rpath=/usr/local/cuda/lib64 > /tmp/lt_ab/$name.log 2>&1 || { echo "variant $name failed"; tail -5 /tmp/lt_ab/$name.log; }

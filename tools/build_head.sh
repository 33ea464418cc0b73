#!/bin/bash
# build the committed (HEAD) libmhd into build/libmhd_prev.so for A/B measurements
set -e
D=$(mktemp -d)
mkdir -p $D/paper_2510_24175_b200/csrc $D/include
SRCS=""
for f in $(git ls-tree --name-only HEAD paper_2510_24175_b200/csrc/); do
  b=$(basename $f); git show HEAD:$f > $D/paper_2510_24175_b200/csrc/$b
  case $b in *.cu) SRCS="$SRCS $b";; esac
done
git show HEAD:include/mhd.h > $D/include/mhd.h
NCCL=$(python -c "import nvidia.nccl as n, os; print(list(n.__path__)[0])")
cd $D/paper_2510_24175_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -shared \
  -I$D/include -I$NCCL/include $SRCS -L$NCCL/lib -l:libnccl.so.2 -Xlinker=-rpath=$NCCL/lib \
  -o $OLDPWD/build/libmhd_prev.so
rm -rf $D

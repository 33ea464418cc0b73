#!/bin/bash
# build the committed (HEAD) libmhd into build/libmhd_prev.so for A/B measurements
set -e
D=$(mktemp -d)
mkdir -p $D/paper_2510_24175_b200/csrc $D/include
for f in mhd_kernels.cu mhd_api.cu mhd_device.cuh mhd_kernels.h; do git show HEAD:paper_2510_24175_b200/csrc/$f > $D/paper_2510_24175_b200/csrc/$f; done
git show HEAD:include/mhd.h > $D/include/mhd.h
NCCL=$(python -c "import nvidia.nccl as n, os; print(list(n.__path__)[0])")
cd $D/paper_2510_24175_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -shared \
  -I$D/include -I$NCCL/include mhd_kernels.cu mhd_api.cu -L$NCCL/lib -l:libnccl.so.2 -Xlinker=-rpath=$NCCL/lib \
  -o $OLDPWD/build/libmhd_prev.so
rm -rf $D

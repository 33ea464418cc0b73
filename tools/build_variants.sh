#!/bin/bash
# build libmhd variants for A/B runs: tools/build_variants.sh name1 "-DA=1 -DB=2" name2 "..." ...
# -> build/libmhd_<name>.so (the in-tree sources with the extra -D flags)
set -e
mkdir -p build
while [ $# -ge 2 ]; do
  n=$1; d=$2; shift 2
  python -m paper_2510_24175_b200.build --out=build/libmhd_$n.so $d > /dev/null &
done
wait
ls -la build/*.so

#!/bin/bash
# A/B of libmhd builds for a scheme: tools/ab_scheme.sh <scheme> lib1.so lib2.so ...
S=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  MHD_LIB=$v timeout 600 python bench.py --scheme $S --steps 6 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ab.log 2>&1
  echo "variant=$v rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1]);print(' value %.4g zu/s  stage %.3f ms' % (d['value'], d['roofline']['stage_ms_per_launch']))" || tail -5 gpurun_out/bench_ab.log
done

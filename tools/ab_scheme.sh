#!/bin/bash
# A/B of libmhd builds on one scheme at 256^3: tools/ab_scheme.sh SCHEME lib1.so lib2.so ...
mkdir -p gpurun_out
sc=$1; shift
for v in "$@"; do
  MHD_LIB=$v timeout 600 python bench.py --workload ot3d --size 256 --scheme $sc --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ab.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1]);print('$sc $v rc=0 value %.4g zu/s  stage %.3f ms' % (d['value'], d['roofline']['stage_ms_per_launch']))" || { echo "$sc $v failed"; tail -3 gpurun_out/bench_ab.log; }
done

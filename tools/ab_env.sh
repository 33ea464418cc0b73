#!/bin/bash
# A/B of environment settings on the 256^3 bench: tools/ab_env.sh "MHD_KZ=86" "MHD_KZ=37" ...
mkdir -p gpurun_out
for v in "$@"; do
  env $v timeout 600 python bench.py --workload ot3d --size 256 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ab.log 2>&1
  echo "setting=$v rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1]);print(' value %.4g zu/s  stage %.3f ms  dt %.3f ms  clocks %s' % (d['value'], d['roofline']['stage_ms_per_launch'], d['roofline']['dt_ms_per_launch'], d['clocks']))" || tail -5 gpurun_out/bench_ab.log
done

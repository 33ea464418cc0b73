#!/bin/bash
# Re-measure everything profiles/ holds, on the GPU box:
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'tools/refresh_profiles.sh r01'
# Writes gpurun_out/<tag>/; copy what is judged into profiles/ afterwards (tools/collect_profiles.sh).
# Order: each ncu capture only after the same command exited 0 without ncu; the one-launch
# stage summaries are written into profiles/ on the box before the bench lines that quote them.
T=${1:-r01}
O=gpurun_out/$T
mkdir -p $O
B="python bench.py"
CELLS=16777216

# 1. PLM stage kernel: plain run, then one full ncu capture (stage 1 of the 4th step)
$B --steps 3 --warmup 3 --no-e2e --no-cpu > $O/plain_plm.log 2>&1 || { echo "plain bench failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:k_stage --launch-skip 6 --launch-count 1 \
  -o $O/ncu_stage_plm $B --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_full_plm.log 2>&1
python tools/ncu_summary.py --json $O/ncu_stage_plm.ncu-rep profiles/ncu_stage_summary.json $CELLS > /dev/null
python tools/ncu_summary.py $O/ncu_stage_plm.ncu-rep > $O/ncu_stage_plm_summary.txt 2>&1
cp profiles/ncu_stage_summary.json $O/

# 2. WENO-Z + RK3 split stage: its x-face kernel (the 10th k_sp_face_x launch = stage 1 of step 4)
$B --scheme wenoz-rk3 --steps 2 --warmup 3 --no-e2e --no-cpu > $O/plain_wz.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:k_sp_face_x --launch-skip 9 --launch-count 1 \
    -o $O/ncu_spx_wenoz $B --scheme wenoz-rk3 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_full_wz.log 2>&1
python tools/ncu_summary.py --json $O/ncu_spx_wenoz.ncu-rep profiles/ncu_stage_summary_wenoz-rk3.json $CELLS \
  "k_sp_face_x of stage 1 (10th launch: after 3 warm-up RK3 steps)" > /dev/null
python tools/ncu_summary.py $O/ncu_spx_wenoz.ncu-rep > $O/ncu_spx_wenoz_summary.txt 2>&1
cp profiles/ncu_stage_summary_wenoz-rk3.json $O/
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_wenoz.csv \
  $B --scheme wenoz-rk3 --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
python tools/launch_share.py $O/launches_wenoz.csv > $O/launch_share_wenoz.txt 2>&1

# 3. launch list of the default bench command (cold-cache, serialised: shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  $B --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu_launch.log 2>&1
python tools/launch_share.py $O/launches.csv > $O/launch_share.txt 2>&1

# 4. bench lines (never under a profiler)
$B > $O/bench.jsonl 2> $O/bench.err
$B --impl reference > $O/bench_reference.jsonl 2> $O/bench_reference.err
$B --workload cpa3d > $O/bench_cpa3d_256.jsonl 2> $O/bench_cpa3d.err
$B --workload blast3d --n 512 --steps 5 --warmup 3 --no-cpu > $O/bench_blast3d_512.jsonl 2> $O/bench_blast3d.err
for sc in wenoz-rk3 ct-plm-rk2 ct-wenoz-rk3; do
  $B --scheme $sc > $O/bench_$sc.jsonl 2> $O/bench_$sc.err
done
$B --n 1024 --steps 3 --warmup 3 --no-cpu --no-e2e > $O/bench_ot3d_1024.jsonl 2> $O/bench_ot3d_1024.err
ls -la $O

#!/bin/bash
# Round-2 measurement set, on the GPU box (one gpurun call; ~15 min):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/refresh_profiles_r02.sh r02'
# Every ncu capture follows a plain run of the same command that exited 0.  Writes gpurun_out/<tag>/
# and the per-stage summaries bench.py quotes (profiles/ncu_stage_<scheme>_<wl><n>.json).
T=${1:-r02}
O=gpurun_out/$T
R=/tmp/ncu_$T   # full reports stay on the box (gpurun brings back <= 64 MiB); summaries go to $O
mkdir -p $O $R
B="python bench.py"
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo "build failed"; exit 1; }

capture() {  # name, cells, bench args...
  local name=$1 cells=$2; shift 2
  $B "$@" --steps 2 --no-e2e --no-cpu > $O/plain_$name.log 2>&1 || { echo "plain $name failed"; return 1; }
  ncu --set full --clock-control none $SRC -k regex:k_stage --launch-skip 6 --launch-count 2 \
    -o $R/ncu_stage_$name $B "$@" --steps 1 --no-e2e --no-cpu > $O/ncu_stage_$name.log 2>&1
  ncu --set full --clock-control none -k regex:k_dt --launch-skip 3 --launch-count 1 \
    -o $R/ncu_dt_$name $B "$@" --steps 1 --no-e2e --no-cpu > $O/ncu_dt_$name.log 2>&1
  python tools/ncu_stage_json.py $R/ncu_stage_$name.ncu-rep $R/ncu_dt_$name.ncu-rep \
    profiles/ncu_stage_plm-rk2_$name.json $cells > /dev/null
  python tools/ncu_summary.py $R/ncu_stage_$name.ncu-rep $R/ncu_dt_$name.ncu-rep > $O/ncu_summary_$name.txt 2>&1
  ncu -i $R/ncu_stage_$name.ncu-rep --page source --csv --print-source sass > $R/sass_$name.csv 2>/dev/null &&
    gzip -c $R/sass_$name.csv > $O/ncu_stage_${name}_sass.csv.gz
  cp profiles/ncu_stage_plm-rk2_$name.json $O/
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$name.csv \
    $B "$@" --steps 2 --no-e2e --no-cpu > /dev/null 2>&1
  python tools/launch_share.py $O/launches_$name.csv > $O/launch_share_$name.txt 2>&1
}
# 1. the default command (weak, configs[3] blast 512^3) and the roofline workload (configs[2] OT 256^3,
#    with source counters)
SRC="" capture blast3d512 134217728
SRC="--import-source on" capture ot3d256 16777216 --workload ot3d --size 256

# 2. WENO-Z + RK3 split stage: its x-face kernel and the launch list
$B --workload ot3d --size 256 --scheme wenoz-rk3 --steps 2 --no-e2e --no-cpu > $O/plain_wz.log 2>&1 &&
  ncu --set full --clock-control none -k regex:k_sp_face_x --launch-skip 9 --launch-count 1 \
    -o $R/ncu_spx_wenoz $B --workload ot3d --size 256 --scheme wenoz-rk3 --steps 1 --no-e2e --no-cpu > $O/ncu_full_wz.log 2>&1
python tools/ncu_summary.py $R/ncu_spx_wenoz.ncu-rep > $O/ncu_spx_wenoz_summary.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches_wenoz.csv $B --workload ot3d --size 256 --scheme wenoz-rk3 --steps 2 --no-e2e --no-cpu > /dev/null 2>&1
python tools/launch_share.py $O/launches_wenoz.csv > $O/launch_share_wenoz.txt 2>&1

# 3. bench lines (never under a profiler)
$B > $O/bench.jsonl 2> $O/bench.err
$B --impl reference > $O/bench_reference.jsonl 2> $O/bench_reference.err
$B --workload ot3d --size 256 > $O/bench_ot3d_256.jsonl 2> $O/bench_ot3d_256.err
$B --scaling strong --steps 3 --no-cpu > $O/bench_strong_1024.jsonl 2> $O/bench_strong_1024.err
$B --workload cpa3d --size 256 --no-cpu > $O/bench_cpa3d_256.jsonl 2> $O/bench_cpa3d.err
for sc in wenoz-rk3 ct-plm-rk2 ct-wenoz-rk3; do
  $B --workload ot3d --size 256 --scheme $sc --no-cpu > $O/bench_$sc.jsonl 2> $O/bench_$sc.err
done
# the roofline workload's stage capture (source counters) comes back if it fits
[ $(stat -c %s $R/ncu_stage_ot3d256.ncu-rep) -lt 40000000 ] && cp $R/ncu_stage_ot3d256.ncu-rep $O/
ls -la $O; du -sh gpurun_out

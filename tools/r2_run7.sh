MHD_LIB=build/libmhd_spxupd.so timeout 600 python -m pytest tests -m gpu -q -x -k "wenoz or random or rare_event" > gpurun_out/r2_gputest7_spxupd.log 2>&1; echo rc=$? >> gpurun_out/r2_gputest7_spxupd.log
MHD_LIB=build/libmhd_fc2p.so timeout 600 python -m pytest tests -m gpu -q -x -k "ot3d or random or rare_event or exact or slab" > gpurun_out/r2_gputest7_fc2p.log 2>&1; echo rc=$? >> gpurun_out/r2_gputest7_fc2p.log
for r in 1 2; do tools/ab.sh build/libmhd_cur2.so build/libmhd_fc2p.so; done > gpurun_out/ab_fc2p.txt 2>&1
for L in build/libmhd_cur2.so build/libmhd_spxupd.so; do
  MHD_LIB=$L python bench.py --workload ot3d --n 256 --scheme wenoz-rk3 --steps 5 --no-e2e --no-cpu > gpurun_out/wz7_$(basename $L).jsonl 2>&1
done

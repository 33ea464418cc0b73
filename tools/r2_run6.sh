python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build6.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -k "wenoz or random or rare_event" > gpurun_out/r2_gputest6.log 2>&1; echo rc=$? >> gpurun_out/r2_gputest6.log
tools/ab.sh build/libmhd_cur.so build/libmhd_wi_nohalo.so build/libmhd_wi_nozconv.so build/libmhd_wi_noupd.so build/libmhd_wi_nopf.so > gpurun_out/ab_wi.txt 2>&1
for L in build/libmhd_prev.so paper_2510_24175_b200/libmhd.so; do
  MHD_LIB=$L python bench.py --workload ot3d --n 256 --scheme wenoz-rk3 --steps 5 --no-e2e --no-cpu > gpurun_out/wz_$(basename $L).jsonl 2>&1
  MHD_LIB=$L ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_sp_face_x --launch-skip 9 --launch-count 1 python bench.py --workload ot3d --n 256 --scheme wenoz-rk3 --steps 1 --no-e2e --no-cpu > gpurun_out/wz_ncu_$(basename $L).txt 2>&1
done

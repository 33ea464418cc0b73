MHD_LIB=build/libmhd_zst.so timeout 600 python -m pytest tests -m gpu -q -x -k "ot3d or random or rare_event or exact or slab or blast or smallest" > gpurun_out/r2_gputest8_zst.log 2>&1; echo rc=$? >> gpurun_out/r2_gputest8_zst.log
for r in 1 2; do tools/ab.sh build/libmhd_cur2.so build/libmhd_zst.so build/libmhd_zstl.so; done > gpurun_out/ab_zst.txt 2>&1

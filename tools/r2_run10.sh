MHD_LIB=build/libmhd_qy.so timeout 700 python -m pytest tests -m gpu -q -x -k "ot2d or ot3d or random or rare_event or exact or slab or smallest or outflow or mixed" > gpurun_out/r2_gputest10_qy.log 2>&1; echo rc=$? >> gpurun_out/r2_gputest10_qy.log
MHD_LIB=build/libmhd_fxo.so timeout 700 python -m pytest tests -m gpu -q -x -k "wenoz or ct or random or rare_event or exact or face_flux" > gpurun_out/r2_gputest10_fxo.log 2>&1; echo rc=$? >> gpurun_out/r2_gputest10_fxo.log
for r in 1 2; do tools/ab.sh build/libmhd_base3.so build/libmhd_qy.so; done > gpurun_out/ab_qy.txt 2>&1
for sc in wenoz-rk3 ct-plm-rk2 ct-wenoz-rk3; do for L in build/libmhd_head3.so build/libmhd_fxi.so build/libmhd_fxo.so; do
  MHD_LIB=$L python bench.py --workload ot3d --n 256 --scheme $sc --steps 5 --no-e2e --no-cpu > gpurun_out/sc10_${sc}_$(basename $L).jsonl 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/sc10_${sc}_$(basename $L).jsonl').read().strip().splitlines()[-1]);print('$sc $L', d['value'], d['roofline']['stage_ms_per_launch'])" >> gpurun_out/ab_fx.txt 2>&1
done; done

mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_2sm -s 1 -c 1 -o gpurun_out/r2r_pair_m2048 python tools/profile_pair.py --m 2048 > gpurun_out/r2r_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_2sm -s 1 -c 1 -o gpurun_out/r2r_pair_m512 python tools/profile_pair.py --m 512 > gpurun_out/r2r_ncu512.log 2>&1

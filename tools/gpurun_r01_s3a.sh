mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:w6a16 -s 2 -c 1 -o gpurun_out/prof_70b_gateup_m16_r5 python tools/profile_one.py --n 57344 --k 8192 --m 16 > gpurun_out/ncu_full.log 2>&1

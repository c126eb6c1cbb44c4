mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:w6a16_tcgen05 -s 2 -c 1 -o gpurun_out/r3s_gateup_m16 python tools/profile_pair.py --n 57344 --k 8192 --m 16 --sched auto > gpurun_out/r3s_ncu.log 2>&1

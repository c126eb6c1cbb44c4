mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:w6a16 -s 2 -c 1 -o gpurun_out/prof_prefill_m2048 python tools/profile_one.py --n 10240 --k 8192 --m 2048 > gpurun_out/ncu_pf.log 2>&1

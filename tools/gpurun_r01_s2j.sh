mkdir -p gpurun_out
timeout 60 ./build/pipe_bench > gpurun_out/pipe_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:w6a16 -s 2 -c 1 -o gpurun_out/prof_70b_down_m16_v3 python tools/profile_one.py --n 8192 --k 28672 --m 16 > gpurun_out/ncu_full.log 2>&1

mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:w6a16 -s 4 -c 4 -o gpurun_out/prof_step7b python tools/profile_step.py > gpurun_out/ncu_step.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:w6a16 -s 4 -c 4 -o gpurun_out/prof_step70b python tools/profile_step.py --model llama2-70b > gpurun_out/ncu_step70.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --burn-in 0 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1

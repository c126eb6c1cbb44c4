#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_v8.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_v8.log
timeout 600 python bench.py --model llama2-70b --steps 500 > gpurun_out/bench70_v8.log 2>&1; echo "bench exit $?" >> gpurun_out/bench70_v8.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_v8.csv python bench.py --steps 20 --warmup 3 --burn-in 0 --no-cpu-baseline > gpurun_out/ncu_launch_v8.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:w6a16 -s 4 -c 4 -o gpurun_out/prof_step7b_v8 python tools/profile_step.py > gpurun_out/ncu_step_v8.log 2>&1
tail -2 gpurun_out/bench_v8.log | cut -c1-600; tail -2 gpurun_out/bench70_v8.log | cut -c1-400

mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 500 --warmup 10 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 600 python bench.py --steps 200 --warmup 10 --model llama2-70b --no-cpu-baseline > gpurun_out/bench70.log 2>&1; echo "bench exit $?" >> gpurun_out/bench70.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --burn-in 0 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:w6a16 -s 2 -c 1 -o gpurun_out/prof_gateup_m16_r3 python tools/profile_one.py --n 22016 --k 4096 --m 16 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:w6a16 -s 2 -c 1 -o gpurun_out/prof_o_m16_r3 python tools/profile_one.py --n 4096 --k 4096 --m 16 > gpurun_out/ncu_full2.log 2>&1

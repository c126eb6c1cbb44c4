set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/probe.py --m 1,16 > gpurun_out/probe.log 2>&1; echo "probe exit $?" >> gpurun_out/probe.log
timeout 600 python bench.py --steps 500 --warmup 10 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --burn-in 0 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:w6a16 -s 2 -c 1 -o gpurun_out/prof_gateup_m16 python tools/profile_one.py --n 22016 --k 4096 --m 16 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:w6a16 -s 2 -c 1 -o gpurun_out/prof_70b_down_m16 python tools/profile_one.py --n 8192 --k 28672 --m 16 > gpurun_out/ncu_full2.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench.log

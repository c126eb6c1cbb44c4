#!/bin/bash
# Round-2 final measurement pass (run via gpurun from the repo root).
TAG=${1:-r02final}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi_$TAG.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_$TAG.log
timeout 600 python bench.py --model llama2-7b --no-cpu-baseline > gpurun_out/bench7_$TAG.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:w6a16 -s 4 -c 4 \
    -o gpurun_out/prof_step70b_$TAG python tools/profile_step.py --model llama2-70b > gpurun_out/ncu_step_$TAG.log 2>&1
tail -2 gpurun_out/pytest_gpu_$TAG.log; tail -2 gpurun_out/bench_$TAG.log | cut -c1-300

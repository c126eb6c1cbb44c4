#!/bin/bash
# One measurement pass on a B200 box (run via gpurun from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- bash tools/gpurun_round.sh TAG
# parity tests, the bench lines (7B default + 70B), the launch list of the
# bench command and one ncu --set full capture of the 7B step; outputs in
# gpurun_out/, summarised into profiles/ with tools/ncu_summary.py.
TAG=${1:-round}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_$TAG.log
timeout 600 python bench.py --model llama2-70b --steps 500 > gpurun_out/bench70_$TAG.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 20 --warmup 3 --burn-in 0 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:w6a16 -s 4 -c 4 \
    -o gpurun_out/prof_step7b_$TAG python tools/profile_step.py > gpurun_out/ncu_step_$TAG.log 2>&1
tail -2 gpurun_out/pytest_gpu_$TAG.log; tail -2 gpurun_out/bench_$TAG.log | cut -c1-400

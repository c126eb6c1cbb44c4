mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --steps 300 > gpurun_out/r3y_bench.log 2>&1; echo "exit $?" >> gpurun_out/r3y_bench.log

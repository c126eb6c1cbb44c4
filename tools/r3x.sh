mkdir -p gpurun_out
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r3x_ref.log 2>&1; echo "exit $?" >> gpurun_out/r3x_ref.log

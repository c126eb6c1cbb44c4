mkdir -p gpurun_out
./build/dq_bench > gpurun_out/r3q_dq_bench.txt 2>&1

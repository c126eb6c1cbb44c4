mkdir -p gpurun_out
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
LPQT_LIB=build/variants/lib_trace.so timeout 120 python tools/chain_trace.py --graph > gpurun_out/chain.log 2>&1

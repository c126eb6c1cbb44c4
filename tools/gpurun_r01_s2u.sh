mkdir -p gpurun_out
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 600 python tools/probe.py --shapes 70b --m 128,512,2048,8192 > gpurun_out/probe_prefill.log 2>&1; echo "probe exit $?" >> gpurun_out/probe_prefill.log

mkdir -p gpurun_out
timeout 600 python tools/probe.py --shapes 7b,70b --m 32,48,64,96 --sched pair > gpurun_out/r3g_probe_pair_m32_96.jsonl 2>&1
timeout 600 python tools/probe.py --shapes 7b,70b --m 32,48,64,96 --sched single > gpurun_out/r3g_probe_single_m32_96.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3g_gpu_tests.log 2>&1; echo "exit $?" >> gpurun_out/r3g_gpu_tests.log

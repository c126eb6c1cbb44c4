mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pair.py -q -x > gpurun_out/r3b_pair_tests.log 2>&1; echo "exit $?" >> gpurun_out/r3b_pair_tests.log
timeout 900 python tools/probe.py --shapes 70b --m 512,2048,8192 > gpurun_out/r3b_probe_prefill.jsonl 2>&1
timeout 600 python tools/probe.py --shapes 7b,13b --m 256,512,1024 > gpurun_out/r3b_probe_prefill_7b13b.jsonl 2>&1

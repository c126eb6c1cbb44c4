mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pair.py -q -x > gpurun_out/r3d_pair_tests.log 2>&1; echo "exit $?" >> gpurun_out/r3d_pair_tests.log
timeout 900 python tools/probe.py --shapes 70b --m 512,2048,8192 > gpurun_out/r3d_probe_prefill.jsonl 2>&1

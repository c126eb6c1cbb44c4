mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_shapes.py -q -x > gpurun_out/r3t_tests.log 2>&1; echo "exit $?" >> gpurun_out/r3t_tests.log
timeout 1500 python tools/probe.py --shapes 7b,13b,sc15b,70b --m 1,2,4,8,16,32,64,128,256,512 > gpurun_out/r3t_probe_all.jsonl 2>&1
timeout 900 python tools/probe.py --shapes 70b --m 1024,2048,4096,8192 > gpurun_out/r3t_probe_70b_big.jsonl 2>&1

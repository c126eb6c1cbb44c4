mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pair.py -q -x -k "fgq or pair" > gpurun_out/r3u_tests.log 2>&1; echo "exit $?" >> gpurun_out/r3u_tests.log
timeout 300 python tools/fgq_bench.py --block 128 --m 512,2048 --shapes 12288x4096,57344x8192,8192x28672 > gpurun_out/r3u_fgq_prefill.jsonl 2>&1
timeout 600 python tools/probe.py --shapes 70b --m 512,2048 > gpurun_out/r3u_probe_70b.jsonl 2>&1

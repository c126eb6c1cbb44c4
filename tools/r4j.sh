mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fp5_native.py tests/test_gpu_fuzz.py tests/test_gpu_pair.py -q -x > gpurun_out/r4j_tests.log 2>&1; echo "exit $?" >> gpurun_out/r4j_tests.log
timeout 300 python tools/fp5_bench.py --m 512,2048 --shapes 70b > gpurun_out/r4j_fp5_prefill.jsonl 2>&1

mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "division_free" > gpurun_out/r4c_selftest.log 2>&1; echo "exit $?" >> gpurun_out/r4c_selftest.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r4c_gpu_tests.log 2>&1; echo "exit $?" >> gpurun_out/r4c_gpu_tests.log
timeout 300 python tools/quant_bench.py --shapes 57344x8192,8192x28672,12288x4096,4096x4096 > gpurun_out/r4c_quant.jsonl 2>&1

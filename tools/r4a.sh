mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_shapes.py tests/test_reference_suite.py -q -x -k "quant or golden or shape or reference or fgq" > gpurun_out/r4a_tests.log 2>&1; echo "exit $?" >> gpurun_out/r4a_tests.log
timeout 300 python tools/quant_bench.py --shapes 57344x8192,8192x28672,12288x4096,4096x4096 > gpurun_out/r4a_quant_fused.jsonl 2>&1
LPQT_LIB=build/variants/lib_twopass.so timeout 300 python tools/quant_bench.py --shapes 57344x8192,8192x28672,12288x4096,4096x4096 > gpurun_out/r4a_quant_twopass.jsonl 2>&1

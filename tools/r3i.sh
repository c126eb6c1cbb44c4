mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ablation.py tests/test_gpu_fp5_native.py -q -x > gpurun_out/r3i_new_tests.log 2>&1; echo "exit $?" >> gpurun_out/r3i_new_tests.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r3i_gpu_tests.log 2>&1; echo "exit $?" >> gpurun_out/r3i_gpu_tests.log

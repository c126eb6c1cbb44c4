mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fuzz.py -q > gpurun_out/r4e_fuzz.log 2>&1; echo "exit $?" >> gpurun_out/r4e_fuzz.log

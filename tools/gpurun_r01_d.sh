mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or linear" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/probe.py --m 16 > gpurun_out/probe_wait2.log 2>&1
LPQT_LIB=build/variants/lib_wait0.so timeout 300 python tools/probe.py --m 16 > gpurun_out/probe_wait0.log 2>&1
LPQT_LIB=build/variants/lib_wait1.so timeout 300 python tools/probe.py --m 16 > gpurun_out/probe_wait1.log 2>&1

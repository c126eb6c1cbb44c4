mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/probe.py --m 1,16 > gpurun_out/probe.log 2>&1
LPQT_LIB=build/variants/lib_trace.so timeout 120 python tools/trace_run.py --n 22016 --k 4096 --m 16 > gpurun_out/trace_gateup.log 2>&1

mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
LPQT_DQG=2 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemm or linear" > gpurun_out/pytest_gpu_dqg2.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_dqg2.log
timeout 400 python tools/probe.py --m 1,16 > gpurun_out/probe_dqg1.log 2>&1
LPQT_DQG=2 timeout 400 python tools/probe.py --m 1,16 > gpurun_out/probe_dqg2.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
tail -2 gpurun_out/pytest_gpu.log gpurun_out/pytest_gpu_dqg2.log

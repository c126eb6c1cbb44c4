mkdir -p gpurun_out
timeout 300 python tools/grid_check.py 8192 8192 1,16,48,100,200,600 0 > gpurun_out/grid.log 2>&1
timeout 300 python tools/grid_check.py 57344,8192 8192,28672 16,100 0 >> gpurun_out/grid.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/probe.py --m 1,16 > gpurun_out/probe.log 2>&1

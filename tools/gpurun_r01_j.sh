mkdir -p gpurun_out
timeout 300 python tools/grid_check.py 2048,4096,8192 2048,8192 100 0,1 > gpurun_out/grid.log 2>&1
timeout 200 python tools/grid_check.py 8192 8192 100,200,600 0 >> gpurun_out/grid.log 2>&1

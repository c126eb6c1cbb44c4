mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r5r_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r5r_pytest.log

mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tp_fused.py tests/test_tp_nccl.py -x -q > gpurun_out/r5v_tp.log 2>&1; echo "rc=$?" >> gpurun_out/r5v_tp.log

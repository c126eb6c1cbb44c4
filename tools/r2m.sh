mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_pair.py -q -x > gpurun_out/r2m_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2m_pytest.log
timeout 300 python tools/probe.py --shapes 70b --m 512,2048,8192 > gpurun_out/r2m_probe.log 2>&1

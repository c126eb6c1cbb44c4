mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_container.py -q -x -k "fgq or container" > gpurun_out/r3m_tests.log 2>&1; echo "exit $?" >> gpurun_out/r3m_tests.log
timeout 300 python tools/fp5_bench.py --m 1,16 --shapes 70b > gpurun_out/r3m_fp5_70b.jsonl 2>&1
timeout 300 python tools/fp5_bench.py --m 1,16 --shapes 7b > gpurun_out/r3m_fp5_7b.jsonl 2>&1
timeout 300 python -m pytest tests/test_gpu_fp5_native.py -q -x > gpurun_out/r3m_fp5_tests.log 2>&1; echo "exit $?" >> gpurun_out/r3m_fp5_tests.log

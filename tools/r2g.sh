mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "fgq or block_params or fp5 or exact or gather or fused" > gpurun_out/r2g_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2g_pytest.log
python tools/fgq_bench.py --m 1,16,32,2048 > gpurun_out/r2g_fgq_bench.log 2>&1

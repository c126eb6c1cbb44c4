mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fgq or block_params or fp5" > gpurun_out/r2i_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2i_pytest.log
python tools/fgq_bench.py --m 1,16,32,64,2048 --shapes 57344x8192,8192x28672,12288x4096,4096x4096 > gpurun_out/r2i_fgq.log 2>&1

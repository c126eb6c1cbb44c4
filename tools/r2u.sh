mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_pair.py tests/test_gpu_parity.py -q -x -k "pair or prefill or gemm_llama or cluster or fgq" > gpurun_out/r2u_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2u_pytest.log
timeout 900 python bench.py > gpurun_out/r2u_bench.log 2>&1

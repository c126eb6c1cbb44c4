mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r6i_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r6i_pytest.log
timeout 1500 python tools/fuzz_big.py 11 200 > gpurun_out/r6i_fuzz_big.jsonl 2>&1; echo "rc=$?" >> gpurun_out/r6i_fuzz_big.jsonl

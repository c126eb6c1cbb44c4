mkdir -p gpurun_out
timeout 1500 python tools/fuzz_big.py 7 200 > gpurun_out/r6h_fuzz_big.jsonl 2>&1; echo "rc=$?" >> gpurun_out/r6h_fuzz_big.jsonl

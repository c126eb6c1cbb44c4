mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "prepack or planes or container or parity or fp5 or exact or baseline" > gpurun_out/r4f_tests.log 2>&1; echo "exit $?" >> gpurun_out/r4f_tests.log
timeout 300 python tools/quant_bench.py --shapes 57344x8192,8192x28672,12288x4096,4096x4096 > gpurun_out/r4f_quant.jsonl 2>&1

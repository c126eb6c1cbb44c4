#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_cli.py tests/test_container.py -x -q > gpurun_out/cli_tests.log 2>&1; echo "rc=$?" >> gpurun_out/cli_tests.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
rm -f gpurun_out/cli_bench.txt
for p in ffn1-1b ffn2-1b ffn1-13b ffn2-13b ffn1-65b ffn2-65b; do timeout 300 python -m paper_2312_08583_b200.cli bench --preset $p --repeat 20 >> gpurun_out/cli_bench.txt 2>&1; done
tail -3 gpurun_out/cli_tests.log; tail -2 gpurun_out/gpu_tests.log; cat gpurun_out/cli_bench.txt

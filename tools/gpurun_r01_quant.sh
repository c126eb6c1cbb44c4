#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "quantize or prepack or encode or empty" > gpurun_out/quant_tests.log 2>&1; echo "quant tests rc=$?" >> gpurun_out/quant_tests.log
timeout 300 python tools/quant_bench.py > gpurun_out/quant_bench.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "all gpu tests rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/quant_tests.log; cat gpurun_out/quant_bench.log; tail -3 gpurun_out/gpu_tests.log

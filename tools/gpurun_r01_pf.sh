#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "prefetch" > gpurun_out/pf_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pf_tests.log
timeout 300 python tools/pf_bench.py --model 7b > gpurun_out/pf_7b.log 2>&1
timeout 300 python tools/pf_bench.py --model 70b > gpurun_out/pf_70b.log 2>&1
timeout 300 python tools/pf_bench.py --model 7b --m 1 --depths -1,32768,65536,131072 > gpurun_out/pf_7b_m1.log 2>&1
tail -3 gpurun_out/pf_tests.log; cat gpurun_out/pf_7b.log gpurun_out/pf_70b.log gpurun_out/pf_7b_m1.log

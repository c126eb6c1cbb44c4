#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python tools/abx.py --libs build/variants/lib_head.so,paper_2312_08583_b200/liblpqt_b200.so --shapes 4096x11008,12288x4096,4096x4096,22016x4096,8192x28672,57344x8192,10240x8192,8192x8192 --m 16 > gpurun_out/abx_fix.log 2>&1
timeout 300 python tools/abx.py --libs build/variants/lib_head.so,paper_2312_08583_b200/liblpqt_b200.so --shapes 4096x11008,8192x28672,4096x4096 --m 1,4,32 > gpurun_out/abx_fix_m.log 2>&1
timeout 300 python tools/pf_bench.py --model 7b --depths=-1,32768,65536 > gpurun_out/pf_7b.log 2>&1
LPQT_LIB=build/variants/lib_trace.so timeout 120 python tools/chain_trace.py --graph > gpurun_out/chain_fix.log 2>&1
tail -2 gpurun_out/gpu_tests.log; cat gpurun_out/abx_fix.log gpurun_out/abx_fix_m.log gpurun_out/pf_7b.log; head -6 gpurun_out/chain_fix.log; grep -A7 "4096, 11008" gpurun_out/chain_fix.log
LPQT_LIB=build/variants/lib_trace.so timeout 120 python tools/chain_trace.py --graph --shapes 4096x11008 > gpurun_out/chain_down.log 2>&1
cat gpurun_out/chain_down.log

#!/bin/bash
mkdir -p gpurun_out
A=paper_2312_08583_b200/liblpqt_b200.so; B=build/variants/lib_bn192.so
timeout 60 python tools/abx.py --libs $B --shapes 4096x4096 --m 512 --rounds 1 --launches 3 > gpurun_out/bn192_smoke.log 2>&1 || { echo "bn192 smoke failed"; cat gpurun_out/bn192_smoke.log; exit 1; }
timeout 600 python tools/abx.py --libs $A,$B --shapes 10240x8192,8192x8192,57344x8192,8192x28672 --m 512,2048,8192 --launches 6 --rounds 3 > gpurun_out/abx_bn192.log 2>&1
cat gpurun_out/abx_bn192.log

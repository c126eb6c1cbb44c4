#!/bin/bash
mkdir -p gpurun_out
A=paper_2312_08583_b200/liblpqt_b200.so; B=build/variants/lib_mma1.so
timeout 60 python tools/abx.py --libs $B --shapes 4096x4096 --m 16 --rounds 1 > gpurun_out/abx_mma1_smoke.log 2>&1 || { echo "mma1 smoke failed/hung"; cat gpurun_out/abx_mma1_smoke.log; exit 1; }
timeout 300 python tools/abx.py --libs $A,$B --shapes 12288x4096,4096x4096,22016x4096,4096x11008,10240x8192,8192x8192,57344x8192,8192x28672 --m 1,16,32 > gpurun_out/abx_mma1.log 2>&1
cat gpurun_out/abx_mma1.log

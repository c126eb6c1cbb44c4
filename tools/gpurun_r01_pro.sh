#!/bin/bash
mkdir -p gpurun_out
A=build/variants/lib_base.so; B=build/variants/lib_pro.so
timeout 60 python tools/abx.py --libs $B --shapes 4096x4096 --m 16 --rounds 1 --launches 3 > /dev/null 2>&1 || { echo "pro smoke failed"; exit 1; }
timeout 600 python tools/abx.py --libs $A,$B --shapes 12288x4096,4096x4096,22016x4096,4096x11008,10240x8192,8192x8192,57344x8192,8192x28672 --m 1,16,128 --rounds 5 > gpurun_out/abx_pro.log 2>&1
cat gpurun_out/abx_pro.log
for L in $A $B; do LPQT_LIB=$L timeout 300 python tools/pf_bench.py --model 7b --depths=-1,65536 --rounds 5; done

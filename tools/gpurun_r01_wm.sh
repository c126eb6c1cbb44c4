#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
A=build/variants/lib_base.so; B=paper_2312_08583_b200/liblpqt_b200.so
timeout 600 python tools/abx.py --libs $A,$B --shapes 12288x4096,4096x4096,22016x4096,4096x11008,10240x8192,8192x8192,57344x8192,8192x28672 --m 1,16,32 --rounds 5 > gpurun_out/abx_wm2.log 2>&1
cat gpurun_out/abx_wm2.log
for L in $A $B; do LPQT_LIB=$L timeout 300 python tools/pf_bench.py --model 7b --depths=65536 --rounds 5; done

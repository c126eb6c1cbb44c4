#!/bin/bash
mkdir -p gpurun_out
A=paper_2312_08583_b200/liblpqt_b200.so; B=build/variants/lib_w1.so; C=build/variants/lib_w3.so; D=build/variants/lib_w4.so
timeout 800 python tools/abx.py --libs $A,$B,$C,$D --shapes 12288x4096,4096x4096,22016x4096,4096x11008,10240x8192,8192x8192,57344x8192,8192x28672 --m 64,128,256,512,2048 --launches 8 --rounds 3 > gpurun_out/abx_wide3.log 2>&1
cat gpurun_out/abx_wide3.log

#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/abx.py --libs paper_2312_08583_b200/liblpqt_b200.so,paper_2312_08583_b200/liblpqt_b200.so,paper_2312_08583_b200/liblpqt_b200.so,paper_2312_08583_b200/liblpqt_b200.so,paper_2312_08583_b200/liblpqt_b200.so,paper_2312_08583_b200/liblpqt_b200.so --flags 0,2,4,4,4,2 --splits 0,0,1,2,3,2 --shapes 12288x4096,4096x4096,22016x4096,4096x11008,10240x8192,8192x8192,57344x8192,8192x28672 --m 1,16 > gpurun_out/sweep.log 2>&1
cat gpurun_out/sweep.log

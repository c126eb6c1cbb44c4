mkdir -p gpurun_out
C=paper_2312_08583_b200/liblpqt_b200.so
timeout 600 python tools/abx.py --libs $C,build/variants/lib_prev.so,$C --flags 2,0,0 --shapes 57344x8192,8192x28672,22016x4096,12288x4096,4096x4096,4096x11008 --m 16 > gpurun_out/abx.log 2>&1
timeout 300 python tools/abx.py --libs $C,$C,$C,$C --flags 2,4,4,4 --splits 0,2,4,8 --shapes 4096x4096,12288x4096,22016x4096 --m 16 >> gpurun_out/abx.log 2>&1
LPQT_LIB=build/variants/lib_trace.so timeout 120 python tools/chain_trace.py --sched cluster --shapes 12288x4096,4096x4096 > gpurun_out/chain.log 2>&1

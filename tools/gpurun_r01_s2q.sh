mkdir -p gpurun_out
rm -f gpurun_out/ab.log
LPQT_LIB=build/variants/lib_prev.so timeout 300 python tools/abbench.py --shapes 8192x28672,22016x4096,4096x4096,57344x8192,12288x4096 --m 16 >> gpurun_out/ab.log 2>&1
timeout 300 python tools/abbench.py --sched streamk --shapes 8192x28672,22016x4096,4096x4096,57344x8192,12288x4096 --m 16 >> gpurun_out/ab.log 2>&1
timeout 300 python tools/abbench.py --sched auto --shapes 22016x4096,4096x4096,12288x4096 --m 16 >> gpurun_out/ab.log 2>&1
LPQT_LIB=build/variants/lib_trace.so timeout 120 python tools/chain_trace.py --sched cluster --shapes 12288x4096,4096x4096 > gpurun_out/chain.log 2>&1
LPQT_LIB=build/variants/lib_trace.so timeout 120 python tools/chain_trace.py --sched auto --shapes 12288x4096,4096x4096 >> gpurun_out/chain.log 2>&1

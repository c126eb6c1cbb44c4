mkdir -p gpurun_out
LPQT_LIB=build/variants/lib_bn64x2.so timeout 900 python tools/sweep_check.py --sets 7b,70b_tp8,ragged --ms 33,48,64 --sched streamk --splits 0,3,7 > gpurun_out/r6d_sweep.jsonl 2>&1
timeout 900 python tools/abx.py --libs build/variants/lib_head7.so,build/variants/lib_bn64x2.so --shapes 10240x8192,8192x8192,57344x8192,8192x28672,12288x4096,4096x4096,22016x4096,4096x11008,1280x8192 --m 33,48,64 --launches 20 --rounds 5 > gpurun_out/r6d_abx.jsonl 2>&1

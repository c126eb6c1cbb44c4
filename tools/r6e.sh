mkdir -p gpurun_out
timeout 900 python tools/abx.py --libs build/variants/lib_head8.so,build/variants/lib_bn64x6.so,build/variants/lib_bn64x8.so --shapes 10240x8192,8192x8192,57344x8192,8192x28672,12288x4096,4096x4096,22016x4096,4096x11008 --m 33,48,64 --launches 20 --rounds 5 > gpurun_out/r6e_abx.jsonl 2>&1

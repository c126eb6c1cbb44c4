mkdir -p gpurun_out
timeout 900 python tools/abx.py --libs build/variants/lib_base.so,build/variants/lib_hint32.so,build/variants/lib_hint128.so --shapes 10240x8192,8192x8192,57344x8192,8192x28672,12288x4096,4096x4096,22016x4096,4096x11008 --m 1,16 --launches 20 --rounds 5 > gpurun_out/r6j_abx_hint.jsonl 2>&1
timeout 900 python tools/abx.py --libs build/variants/lib_base.so,build/variants/lib_hint32.so,build/variants/lib_hint128.so --shapes 8192x8192,57344x8192 --m 512,2048 --launches 5 --rounds 5 >> gpurun_out/r6j_abx_hint.jsonl 2>&1

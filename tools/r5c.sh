mkdir -p gpurun_out
L=paper_2312_08583_b200/liblpqt_b200.so
timeout 900 python tools/abx.py --libs $L,build/variants/lib_b224x8.so --shapes 10240x8192,8192x8192,57344x8192,8192x28672,12288x4096,4096x4096,22016x4096,4096x11008 --m 1,16 --launches 20 --rounds 5 > gpurun_out/r5c_abx_xstages8.jsonl 2>&1

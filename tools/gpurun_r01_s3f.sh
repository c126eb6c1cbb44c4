mkdir -p gpurun_out
C=paper_2312_08583_b200/liblpqt_b200.so
timeout 900 python tools/abx.py --libs $C,build/variants/lib_1iss.so --shapes 57344x8192,8192x28672,22016x4096,12288x4096,4096x4096,4096x11008,10240x8192,8192x8192 --m 16 > gpurun_out/abx_1iss.log 2>&1

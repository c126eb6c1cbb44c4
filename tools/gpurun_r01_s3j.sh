mkdir -p gpurun_out
C=paper_2312_08583_b200/liblpqt_b200.so
timeout 900 python tools/abx.py --libs $C,build/variants/lib_x3.so,build/variants/lib_bn128.so --shapes 10240x8192,57344x8192,8192x28672 --m 512,2048,8192 --launches 6 --rounds 3 > gpurun_out/abx_pf.log 2>&1

mkdir -p gpurun_out
C=paper_2312_08583_b200/liblpqt_b200.so
timeout 900 python tools/abx.py --libs $C,build/variants/lib_nomma.so,build/variants/lib_norebuild.so,build/variants/lib_nonone.so --shapes 57344x8192,8192x28672,22016x4096,4096x4096 --m 16 > gpurun_out/abx_iso.log 2>&1

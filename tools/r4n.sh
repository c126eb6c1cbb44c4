mkdir -p gpurun_out
L=paper_2312_08583_b200/liblpqt_b200.so
timeout 600 python tools/abx.py --libs build/variants/lib_head.so,build/variants/lib_wp4.so,$L,build/variants/lib_wp64.so,build/variants/lib_nowd.so --shapes 10240x8192,8192x8192,57344x8192,8192x28672,12288x4096,4096x4096,22016x4096,4096x11008 --m 16 --launches 20 --rounds 5 > gpurun_out/r4n_abx_wp.jsonl 2>&1
timeout 600 python tools/abx.py --libs build/variants/lib_head.so,build/variants/lib_wp4.so,$L,build/variants/lib_wp64.so,build/variants/lib_nowd.so --shapes 10240x8192,8192x8192,57344x8192,8192x28672 --m 1 --launches 20 --rounds 5 > gpurun_out/r4n_abx_wp_m1.jsonl 2>&1

mkdir -p gpurun_out
L=paper_2312_08583_b200/liblpqt_b200.so
timeout 900 python tools/abx.py --libs build/variants/lib_head3.so,$L --shapes 1280x8192,1024x8192,1024x28672,2560x8192,2048x8192,2048x28672,4096x4096,5120x5120,6144x6144,6400x6144 --m 40,64 --launches 20 --rounds 5 > gpurun_out/r4s_abx_splitcap.jsonl 2>&1

mkdir -p gpurun_out
L=paper_2312_08583_b200/liblpqt_b200.so
timeout 900 python tools/abx.py --libs $L,$L,$L,$L,$L --flags 0,16,8,8,8 --splits 0,2,2,4,8 --shapes 4096x4096,5120x5120,6144x6144,4096x11008,12288x4096,1280x8192,2560x8192 --m 96,128,192,256 --launches 10 --rounds 5 > gpurun_out/r5y_abx_smallprefill.jsonl 2>&1

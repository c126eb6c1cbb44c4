mkdir -p gpurun_out
L=paper_2312_08583_b200/liblpqt_b200.so
timeout 900 python tools/abx.py --libs $L --shapes 10240x8192,8192x8192,57344x8192,12288x4096,4096x4096,5120x13824 --m 16,24,32,33,40,48,64,65,96,128 --launches 20 --rounds 3 > gpurun_out/r5f_abx_m_sweep.jsonl 2>&1

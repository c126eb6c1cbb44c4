mkdir -p gpurun_out
LPQT_LIB=build/variants/lib_csk1y.so timeout 900 python tools/sweep_check.py --sets 7b,70b_tp8,ragged,13b,sc15b --ms 17,24,32 --sched cluster --splits 0,2,3,5 > gpurun_out/r6c_sweep.jsonl 2>&1
timeout 900 python tools/abx.py --libs build/variants/lib_head6.so,build/variants/lib_csk1y.so --shapes 4096x4096,5120x5120,6144x6144,6400x6144 --m 17,24,32 --launches 20 --rounds 5 > gpurun_out/r6c_abx.jsonl 2>&1

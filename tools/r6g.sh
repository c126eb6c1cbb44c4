mkdir -p gpurun_out
L=build/variants/lib_cur.so
timeout 900 python tools/abx.py --libs $L,$L,$L --flags 0,16,16 --splits 0,1,2 --shapes 10240x8192,8192x8192,57344x8192,8192x28672 --m 512,1024,2048 --launches 5 --rounds 5 > gpurun_out/r6g_abx.jsonl 2>&1

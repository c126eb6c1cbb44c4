mkdir -p gpurun_out
python tools/abx.py --libs build/variants/lib_px3.so,build/variants/lib_px4.so --shapes 8192x8192,57344x8192,8192x28672,10240x8192 --m 512,2048,8192 --launches 10 --rounds 3 > gpurun_out/r2k_abx.log 2>&1

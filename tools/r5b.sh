mkdir -p gpurun_out
L=paper_2312_08583_b200/liblpqt_b200.so
LPQT_LIB=build/variants/lib_ks2x2.so timeout 600 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -x -q > gpurun_out/r5b_pytest_ks2.log 2>&1; echo "rc=$?" >> gpurun_out/r5b_pytest_ks2.log
timeout 900 python tools/abx.py --libs $L,build/variants/lib_ks2x2.so --shapes 1280x8192,2560x8192,4096x4096,5120x5120,6144x6144,12288x4096,4096x11008,8192x8192,8192x28672,15360x5120 --m 33,48,64 --launches 20 --rounds 5 > gpurun_out/r5b_abx_ks2.jsonl 2>&1

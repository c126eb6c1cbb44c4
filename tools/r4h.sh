mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pair.py tests/test_gpu_fuzz.py -q -x > gpurun_out/r4h_tests.log 2>&1; echo "exit $?" >> gpurun_out/r4h_tests.log
L=paper_2312_08583_b200/liblpqt_b200.so
timeout 900 python tools/abx.py --libs $L,build/variants/lib_head.so --shapes 4096x4096,5120x5120,6144x6144,12288x4096,10240x8192,8192x8192,57344x8192 --m 128,256,512 --launches 10 --rounds 5 > gpurun_out/r4h_abx_batch.jsonl 2>&1

mkdir -p gpurun_out
LPQT_LIB=build/variants/lib_bn32x2.so timeout 600 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_streamk_fixup.py -x -q > gpurun_out/r5w_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r5w_pytest.log
timeout 900 python tools/abx.py --libs build/variants/lib_head4.so,build/variants/lib_bn32x2.so --shapes 10240x8192,8192x8192,57344x8192,8192x28672,12288x4096,4096x4096,22016x4096,4096x11008,5120x5120,6144x6144 --m 17,24,32 --launches 20 --rounds 5 > gpurun_out/r5w_abx_bn32x.jsonl 2>&1

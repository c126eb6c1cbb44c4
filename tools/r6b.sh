mkdir -p gpurun_out
LPQT_LIB=build/variants/lib_oney.so timeout 600 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_streamk_fixup.py tests/test_gpu_parity.py -x -q > gpurun_out/r6b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r6b_pytest.log
LPQT_LIB=build/variants/lib_oney.so timeout 600 python tools/sweep_check.py --sets 7b,70b,70b_tp8,ragged --ms 17,24,32 --sched streamk --splits 0,3,7 > gpurun_out/r6b_sweep.jsonl 2>&1
timeout 900 python tools/abx.py --libs build/variants/lib_head5.so,build/variants/lib_oney.so --shapes 10240x8192,8192x8192,57344x8192,8192x28672,12288x4096,22016x4096,4096x11008,15360x5120,27648x5120 --m 17,24,32 --launches 20 --rounds 5 > gpurun_out/r6b_abx_oney.jsonl 2>&1

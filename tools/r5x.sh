mkdir -p gpurun_out
L=paper_2312_08583_b200/liblpqt_b200.so
timeout 600 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_streamk_fixup.py tests/test_gpu_parity.py -x -q > gpurun_out/r5x_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r5x_pytest.log
timeout 900 python tools/abx.py --libs $L,$L,$L --flags 0,4,4 --splits 0,2,3 --shapes 10240x8192,8192x8192,57344x8192,8192x28672,12288x4096,22016x4096,4096x11008,4096x4096 --m 24 --launches 20 --rounds 5 > gpurun_out/r5x_abx_csk32.jsonl 2>&1

mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pair.py -q -x > gpurun_out/r3p_pair_tests.log 2>&1; echo "exit $?" >> gpurun_out/r3p_pair_tests.log
L=paper_2312_08583_b200/liblpqt_b200.so
timeout 900 python tools/abx.py --libs $L,build/variants/lib_nosplit.so --shapes 10240x8192,8192x8192,57344x8192,8192x28672,12288x4096,4096x4096,22016x4096,4096x11008 --m 512,2048 --launches 10 --rounds 4 > gpurun_out/r3p_abx_nsplit.jsonl 2>&1
timeout 900 python tools/probe.py --shapes 70b --m 512,2048,8192 > gpurun_out/r3p_probe_70b.jsonl 2>&1

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pair.py -q -x > gpurun_out/r3c_pair_tests.log 2>&1; echo "exit $?" >> gpurun_out/r3c_pair_tests.log
timeout 900 python tools/probe.py --shapes 70b --m 512,2048,8192 > gpurun_out/r3c_probe_prefill.jsonl 2>&1
L=paper_2312_08583_b200/liblpqt_b200.so
timeout 600 python tools/abx.py --libs $L,build/variants/lib_nopro.so --shapes 10240x8192,8192x8192,57344x8192,8192x28672,12288x4096,4096x4096,22016x4096,4096x11008 --m 1,16 --launches 20 --rounds 5 > gpurun_out/r3c_abx_prologue.jsonl 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 500 > gpurun_out/r3c_bench.log 2>&1

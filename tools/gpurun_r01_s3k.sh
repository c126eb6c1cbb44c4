mkdir -p gpurun_out
C=paper_2312_08583_b200/liblpqt_b200.so
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/abx.py --libs $C,build/variants/lib_x3.so --shapes 10240x8192,57344x8192,8192x28672,8192x8192 --m 512,2048,8192 --launches 6 --rounds 3 > gpurun_out/abx_pf.log 2>&1
timeout 600 python tools/probe.py --shapes 70b --m 128,512,2048,8192 > gpurun_out/probe_prefill.log 2>&1

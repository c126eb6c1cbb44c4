mkdir -p gpurun_out
C=paper_2312_08583_b200/liblpqt_b200.so
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python tools/abx.py --libs $C,build/variants/lib_base.so,$C,build/variants/lib_base.so --flags 0,0,2,2 --shapes 57344x8192,8192x28672,22016x4096,12288x4096,4096x4096,4096x11008,10240x8192,8192x8192 --m 16 > gpurun_out/abx_spec.log 2>&1
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log

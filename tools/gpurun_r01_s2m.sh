mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/grid_check.py 4096,22016 4096,11008,384,1000 1,16,17,48,200 0,1,3 > gpurun_out/grid.log 2>&1; echo "grid exit $?" >> gpurun_out/grid.log
rm -f gpurun_out/ab.log
for lib in "" build/variants/lib_natorder.so build/variants/lib_v1.so; do
  LPQT_LIB=$lib timeout 300 python tools/abbench.py --shapes 8192x28672,22016x4096,4096x4096,57344x8192,12288x4096,4096x11008 --m 1,16 >> gpurun_out/ab.log 2>&1
done
timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log

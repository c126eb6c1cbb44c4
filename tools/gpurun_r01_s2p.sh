mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/ab.log
for sc in auto streamk; do
  timeout 300 python tools/abbench.py --sched $sc --shapes 8192x28672,22016x4096,4096x4096,57344x8192,12288x4096,4096x11008,10240x8192,8192x8192 --m 1,16 >> gpurun_out/ab.log 2>&1
done
timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log

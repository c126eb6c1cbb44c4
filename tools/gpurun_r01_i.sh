mkdir -p gpurun_out
rm -f gpurun_out/one.log
cp tools/one_shape.py /tmp/one.py
for s in "12288 4096 1" "4096 4096 16" "22016 4096 16" "4096 11008 16" "10240 8192 16" "8192 8192 1" "57344 8192 16" "8192 28672 1" "8192 28672 48" "8192 8192 100" "8192 8192 600"; do
  timeout 30 python /tmp/one.py $s >> gpurun_out/one.log 2>&1 || echo "FAIL/TIMEOUT $s" >> gpurun_out/one.log
done
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/probe.py --m 1,16 > gpurun_out/probe.log 2>&1

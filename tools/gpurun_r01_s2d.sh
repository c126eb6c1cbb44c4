mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/trace.log
for s in "4096 4096 16" "22016 4096 16" "8192 28672 16" "57344 8192 1"; do
  LPQT_LIB=build/variants/lib_trace.so timeout 120 python tools/trace_run.py --n ${s% * *} --k $(echo $s | cut -d' ' -f2) --m ${s##* } >> gpurun_out/trace.log 2>&1
done
timeout 300 python tools/probe.py --m 1,16 > gpurun_out/probe.log 2>&1; echo "probe exit $?" >> gpurun_out/probe.log
timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log

mkdir -p gpurun_out
timeout 120 ./build/launch_bench > gpurun_out/launch_bench.log 2>&1; echo "exit $?" >> gpurun_out/launch_bench.log
export LPQT_LIB=build/variants/lib_trace.so
for s in "4096 4096 16" "22016 4096 16" "8192 28672 16" "57344 8192 1"; do
  timeout 120 python tools/trace_run.py --n ${s% * *} --k $(echo $s | cut -d' ' -f2) --m ${s##* } --events >> gpurun_out/trace.log 2>&1
done

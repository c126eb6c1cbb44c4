mkdir -p gpurun_out
rm -f gpurun_out/trace.log
for s in "4096 4096 16" "22016 4096 16" "8192 28672 16"; do
  LPQT_LIB=build/variants/lib_trace.so timeout 120 python tools/trace_run.py --n ${s% * *} --k $(echo $s | cut -d' ' -f2) --m ${s##* } >> gpurun_out/trace.log 2>&1
done

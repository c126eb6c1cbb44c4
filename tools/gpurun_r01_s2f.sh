mkdir -p gpurun_out
rm -f gpurun_out/trace.log
for lib in lib_trace lib_trace_nostore; do
for o in f16 f32; do
  LPQT_LIB=build/variants/$lib.so timeout 120 python tools/trace_run.py --n 22016 --k 4096 --m 16 --out $o >> gpurun_out/trace.log 2>&1
done; done

mkdir -p gpurun_out
rm -f gpurun_out/ab.log
for lib in "" build/variants/lib_v1.so; do
  LPQT_LIB=$lib timeout 300 python tools/abbench.py --shapes 8192x28672,22016x4096,4096x4096,57344x8192,12288x4096,4096x11008 --m 1,16 >> gpurun_out/ab.log 2>&1
done

mkdir -p gpurun_out
L=paper_2312_08583_b200/liblpqt_b200.so
timeout 600 python tools/abx.py --libs $L,build/variants/lib_nowd.so,build/variants/lib_wd8.so --shapes 10240x8192,8192x8192,57344x8192,8192x28672,12288x4096,4096x4096,22016x4096,4096x11008 --m 16 --launches 20 --rounds 5 > gpurun_out/r4l_abx_wd.jsonl 2>&1
for v in base nowd wd8; do
  if [ $v == base ]; then unset LPQT_LIB; else export LPQT_LIB=build/variants/lib_$v.so; fi
  timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 1000 > gpurun_out/r4l_bench70_$v.log 2>&1
  timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 1000 --model llama2-7b > gpurun_out/r4l_bench7_$v.log 2>&1
done

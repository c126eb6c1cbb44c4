mkdir -p gpurun_out
L=paper_2312_08583_b200/liblpqt_b200.so
for v in dd1 dd2; do
  LPQT_LIB=build/variants/lib_$v.so timeout 600 python -m pytest tests/test_gpu_pair.py tests/test_gpu_fuzz.py tests/test_gpu_baseline_shapes.py -x -q > gpurun_out/r5e_pytest_$v.log 2>&1; echo "rc=$?" >> gpurun_out/r5e_pytest_$v.log
done
timeout 1200 python tools/abx.py --libs $L,build/variants/lib_dd1.so,build/variants/lib_dd2.so --shapes 12288x4096,4096x4096,22016x4096,4096x11008,10240x8192,8192x8192,57344x8192,8192x28672 --m 512,2048 --launches 5 --rounds 5 > gpurun_out/r5e_abx_dd.jsonl 2>&1

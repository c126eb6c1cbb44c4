mkdir -p gpurun_out
timeout 300 python tools/repro_bn64.py 5120 13824 33,48,64 > gpurun_out/r5g_repro.log 2>&1
echo "rc=$?" >> gpurun_out/r5g_repro.log
timeout 600 compute-sanitizer --tool memcheck --kernel-name kns=w6a16_tcgen05 --print-limit 5 python tools/repro_bn64.py 5120 13824 33 > gpurun_out/r5g_memcheck.log 2>&1
echo "rc=$?" >> gpurun_out/r5g_memcheck.log

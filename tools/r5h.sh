mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_streamk_fixup.py -x -q > gpurun_out/r5h_fixup.log 2>&1; echo "rc=$?" >> gpurun_out/r5h_fixup.log
LPQT_LIB=build/variants/lib_head3.so timeout 600 python -m pytest tests/test_gpu_streamk_fixup.py -q > gpurun_out/r5h_fixup_old.log 2>&1; echo "rc=$?" >> gpurun_out/r5h_fixup_old.log
timeout 300 python tools/repro_bn64.py 5120 13824 33,48,64 > gpurun_out/r5h_repro.log 2>&1

mkdir -p gpurun_out
export LPQT_LIB=build/variants/lib_trace.so
timeout 120 python tools/trace_run.py --n 22016 --k 4096 --m 16 > gpurun_out/trace_gateup.log 2>&1
timeout 120 python tools/trace_run.py --n 4096 --k 4096 --m 16 > gpurun_out/trace_o.log 2>&1
timeout 120 python tools/trace_run.py --n 57344 --k 8192 --m 1 > gpurun_out/trace_70b_gateup.log 2>&1

mkdir -p gpurun_out
export LPQT_LIB=build/variants/lib_trace.so
python tools/chain_trace.py --shapes 10240x8192,8192x8192,57344x8192,8192x28672 --m 16 --graph --pf 0 > gpurun_out/r2d_trace70_graph.txt 2>&1
python tools/chain_trace.py --shapes 10240x8192,8192x8192,57344x8192,8192x28672 --m 16 > gpurun_out/r2d_trace70_eager.txt 2>&1
python tools/chain_trace.py --shapes 12288x4096,4096x4096,22016x4096,4096x11008 --m 16 --graph --pf 0 > gpurun_out/r2d_trace7_graph.txt 2>&1

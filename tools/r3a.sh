mkdir -p gpurun_out
export LPQT_LIB=build/variants/lib_trace.so
python tools/chain_trace.py --shapes 12288x4096,4096x4096,22016x4096,4096x11008 --m 16 --graph --pf 0 > gpurun_out/r3a_trace7_graph.txt 2>&1
python tools/chain_trace.py --shapes 10240x8192,8192x8192,57344x8192,8192x28672 --m 16 --graph --pf 0 > gpurun_out/r3a_trace70_graph.txt 2>&1
python tools/chain_trace.py --shapes 4096x4096 --m 16 --reps 3 > gpurun_out/r3a_trace_o7.txt 2>&1
unset LPQT_LIB
python tools/abx.py --libs paper_2312_08583_b200/liblpqt_b200.so --shapes 12288x4096,4096x4096,22016x4096,4096x11008,10240x8192,8192x8192 --m 1,16 > gpurun_out/r3a_abx_base.jsonl 2>&1

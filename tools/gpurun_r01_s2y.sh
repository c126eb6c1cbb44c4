mkdir -p gpurun_out
rm -f gpurun_out/chain_c.log
for c in 4 8; do
LPQT_LIB=build/variants/lib_trace.so timeout 120 python tools/chain_trace.py --graph --sched cluster --split $c --shapes 4096x4096,4096x4096 >> gpurun_out/chain_c.log 2>&1
done

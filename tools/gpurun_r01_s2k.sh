mkdir -p gpurun_out
rm -f gpurun_out/trace_var.log
for lib in lib_trace lib_no_aempty lib_no_rebuild lib_no_aempty_lpqt_exp_no_rebuild; do
  LPQT_LIB=build/variants/$lib.so timeout 120 python tools/trace_run.py --n 8192 --k 28672 --m 16 > /tmp/t.log 2>&1
  echo "== $lib" >> gpurun_out/trace_var.log; grep -E "shape|prodW|dq0_done|mma_done|epi_done|span" /tmp/t.log >> gpurun_out/trace_var.log
  sed -n '/per-stage clock64/,/DQ warps/p' /tmp/t.log | sed -n 22,26p >> gpurun_out/trace_var.log
done

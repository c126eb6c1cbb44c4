mkdir -p gpurun_out
for v in pd4w0 pd6w0 pd4w1 pd6w1; do
  echo "== $v" >> gpurun_out/r2h_fgq.log
  LPQT_LIB=build/variants/lib_$v.so python tools/fgq_bench.py --m 1,16 --shapes 57344x8192,8192x28672,12288x4096 >> gpurun_out/r2h_fgq.log 2>&1
done
LPQT_LIB=build/variants/lib_pd6w0.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fgq or block_params" > gpurun_out/r2h_pytest6.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2h_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2h_pytest.log

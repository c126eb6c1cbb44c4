mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_pair.py -q -x > gpurun_out/r2o_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2o_pytest.log
for s in pair single; do
for m in 512 2048 8192; do
  python tools/abx.py --libs paper_2312_08583_b200/liblpqt_b200.so --flags $([ $s == pair ] && echo 16 || echo 8) --shapes 8192x8192,57344x8192,8192x28672,10240x8192 --m $m --launches 5 --rounds 2 >> gpurun_out/r2o_abx_$s.log 2>&1
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_2sm -s 1 -c 1 -o gpurun_out/r2o_pair_m2048 python tools/profile_pair.py --m 2048 > gpurun_out/r2o_ncu.log 2>&1

mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_pair.py -q -x > gpurun_out/r2p_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2p_pytest.log
for m in 512 2048 8192; do
  python tools/abx.py --libs paper_2312_08583_b200/liblpqt_b200.so,paper_2312_08583_b200/liblpqt_b200.so --flags 16,8 --shapes 8192x8192,57344x8192,8192x28672,10240x8192 --m $m --launches 5 --rounds 2 >> gpurun_out/r2p_abx.log 2>&1
done
timeout 600 python tools/probe.py --shapes 70b --m 512,2048,8192 > gpurun_out/r2p_probe.log 2>&1

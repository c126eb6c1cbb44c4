mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fgq" > gpurun_out/r3l_fgq_tests.log 2>&1; echo "exit $?" >> gpurun_out/r3l_fgq_tests.log
for b in 128 64 32 16; do timeout 150 python tools/fgq_bench.py --block $b --m 1,16 --shapes 12288x4096,57344x8192,8192x28672 > gpurun_out/r3l_fgq_b$b.jsonl 2>&1; done
timeout 300 python tools/fp5_bench.py --m 1,16 --shapes 70b > gpurun_out/r3l_fp5_70b.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_2sm -s 1 -c 1 -o gpurun_out/r3l_pair_sk_m512 python tools/profile_pair.py --n 10240 --k 8192 --m 512 > gpurun_out/r3l_ncu_sk512.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_2sm -s 1 -c 1 -o gpurun_out/r3l_pair_gu_m512 python tools/profile_pair.py --n 57344 --k 8192 --m 512 > gpurun_out/r3l_ncu_gu512.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r3l_gpu_tests.log 2>&1; echo "exit $?" >> gpurun_out/r3l_gpu_tests.log

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fgq" > gpurun_out/r3k_fgq_tests.log 2>&1; echo "exit $?" >> gpurun_out/r3k_fgq_tests.log
for b in 128 64 32 16; do timeout 600 python tools/fgq_bench.py --block $b --m 1,16 --shapes 12288x4096,57344x8192,8192x28672 > gpurun_out/r3k_fgq_b$b.jsonl 2>&1; done

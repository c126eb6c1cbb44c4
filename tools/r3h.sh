mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ablation.py -q -x > gpurun_out/r3h_ablation_tests.log 2>&1; echo "exit $?" >> gpurun_out/r3h_ablation_tests.log
timeout 600 python tools/ablation_bench.py --m 8 > gpurun_out/r3h_ablation_paper.jsonl 2>&1
timeout 600 python tools/ablation_bench.py --m 1,16 --shapes 70b > gpurun_out/r3h_ablation_70b.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3h_gpu_tests.log 2>&1; echo "exit $?" >> gpurun_out/r3h_gpu_tests.log

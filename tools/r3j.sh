mkdir -p gpurun_out
timeout 600 python tools/fp5_bench.py --m 1,8,16 --shapes 70b > gpurun_out/r3j_fp5_70b.jsonl 2>&1
timeout 600 python tools/fp5_bench.py --m 1,16 --shapes 7b > gpurun_out/r3j_fp5_7b.jsonl 2>&1
timeout 600 python tools/ablation_bench.py --m 8 > gpurun_out/r3j_ablation_paper.jsonl 2>&1
timeout 600 python tools/ablation_bench.py --m 1,16 --shapes 70b > gpurun_out/r3j_ablation_70b.jsonl 2>&1
timeout 900 python bench.py > gpurun_out/r3j_bench.log 2>&1

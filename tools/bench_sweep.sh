mkdir -p gpurun_out
for cfg in "--graph-steps 1" "--graph-steps 8" "--graph-steps 8 --no-l2-next" "--graph-steps 1" "--graph-steps 8" "--graph-steps 8 --no-l2-next"; do
  echo "== $cfg" >> gpurun_out/r2e_bench.log
  timeout 300 python bench.py --no-extras --no-cpu-baseline $cfg 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['roofline']['frac'], d['ms_per_step'], d['cublas_fp16']['speedup_vs_cublas'], d['clocks'], d['e2e']['value'])" >> gpurun_out/r2e_bench.log
done
for cfg in "--graph-steps 1" "--graph-steps 8" "--graph-steps 8 --no-l2-next"; do
  echo "== 7b $cfg" >> gpurun_out/r2e_bench.log
  timeout 300 python bench.py --model llama2-7b --no-extras --no-cpu-baseline $cfg 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['roofline']['frac'], d['ms_per_step'], d['cublas_fp16']['speedup_vs_cublas'], d['clocks'], d['e2e']['value'])" >> gpurun_out/r2e_bench.log
done

mkdir -p gpurun_out
for g in 8 16 32; do
  timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 1000 --graph-steps $g > gpurun_out/r4k_g$g.log 2>&1
done
for g in 8 16 32; do
  timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 1000 --graph-steps $g > gpurun_out/r4k_g${g}_b.log 2>&1
done

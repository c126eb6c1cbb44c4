mkdir -p gpurun_out
for pf in 0 131072 196608 262144 393216; do
  for mdl in llama2-70b llama2-7b; do
    timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 400 --model $mdl --pf-bytes $pf > gpurun_out/r3o_pf_${mdl}_$pf.log 2>&1
  done
done

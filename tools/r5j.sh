mkdir -p gpurun_out
for kind in fgq128 fgq64 fgq16 fp5; do
  timeout 900 python tools/sweep_check.py --kind $kind --sets 7b,70b,70b_tp8 > gpurun_out/r5j_sweep_$kind.jsonl 2>&1; echo "rc=$?" >> gpurun_out/r5j_sweep_$kind.jsonl
done

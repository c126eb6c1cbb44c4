mkdir -p gpurun_out
for kind in int4 int4_128; do
  timeout 900 python tools/sweep_check.py --kind $kind --sets 7b,70b_tp8 > gpurun_out/r5l_sweep_$kind.jsonl 2>&1; echo "rc=$?" >> gpurun_out/r5l_sweep_$kind.jsonl
done

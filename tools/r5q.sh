mkdir -p gpurun_out
O=gpurun_out/r5q_sweeps_bigm.jsonl; : > $O
for kind in cgq fgq128 fp5 int4_128; do
  timeout 900 python tools/sweep_check.py --sets 70b,ragged --kind $kind --ms 2048,4096,8192 | tail -1 >> $O 2>&1
done

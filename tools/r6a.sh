mkdir -p gpurun_out
O=gpurun_out/r6a_sweeps_csk32.jsonl; : > $O
for kind in cgq fgq128 fgq16 fp5 int4_128; do
  timeout 900 python tools/sweep_check.py --sets 7b,70b,70b_tp8,ragged,13b --kind $kind --sched cluster --splits 0,2,3,5,8 --ms 17,24,32 | tail -1 >> $O 2>&1
done
timeout 900 python tools/sweep_check.py --sets 7b,70b,70b_tp8,ragged,13b,sc15b --ms 17,20,24,28,32 | tail -1 >> $O 2>&1

mkdir -p gpurun_out
O=gpurun_out/r5t_sweeps_ablation.jsonl; : > $O
for rb in bias_shift naive; do
  timeout 900 python tools/sweep_check.py --sets 7b,70b_tp8,ragged --rebuild $rb --ms 1,8,16 | tail -1 >> $O 2>&1
  timeout 900 python tools/sweep_check.py --sets 7b,ragged --rebuild $rb --sched cluster --splits 2,3 --ms 1,16 | tail -1 >> $O 2>&1
  timeout 900 python tools/sweep_check.py --sets 7b,ragged --rebuild $rb --sched streamk --splits 3,7 --ms 1,16 | tail -1 >> $O 2>&1
done

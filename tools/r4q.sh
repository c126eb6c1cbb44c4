mkdir -p gpurun_out
for s in auto single streamk pair; do
  timeout 300 python tools/probe.py --shapes 70b_tp8,70b_tp4 --m 128,256,512 --sched $s > gpurun_out/r4q_tp_$s.jsonl 2>&1
done

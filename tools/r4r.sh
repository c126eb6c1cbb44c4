mkdir -p gpurun_out
for s in single pair; do
  timeout 600 python tools/probe.py --shapes 70b_tp8 --m 64,128,256 --sched $s --split 0,2,4,8,16 > gpurun_out/r4r_tp8_split_$s.jsonl 2>&1
done

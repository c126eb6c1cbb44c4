mkdir -p gpurun_out
O=gpurun_out/r5z_sweeps_oddm.jsonl; : > $O
for kind in cgq fgq128 fp5 int4_128; do
  timeout 900 python tools/sweep_check.py --sets 7b,70b_tp8,ragged --kind $kind --ms 65,97,129,191,257,300,511,513,700,1000,1023,1025,2049 | tail -1 >> $O 2>&1
done
timeout 900 python tools/sweep_check.py --sets 7b,70b_tp8,ragged --ms 65,97,129,300,700,1025 --sched pair --splits 1,2 | tail -1 >> $O 2>&1
timeout 900 python tools/sweep_check.py --sets 7b,70b_tp8,ragged --ms 65,97,129,300,700,1025 --layout nm | tail -1 >> $O 2>&1

mkdir -p gpurun_out
O=gpurun_out/r5p2_sweeps.jsonl; : > $O
for kind in fgq128 fgq16 fp5; do
  timeout 600 python tools/sweep_check.py --sets ragged,7b --kind $kind --sched cluster --splits 2,3,5 --ms 1,16,32 | tail -1 >> $O 2>&1
  timeout 600 python tools/sweep_check.py --sets ragged,7b --kind $kind --sched streamk --splits 3,7 --ms 1,16,32,48 | tail -1 >> $O 2>&1
done
for out in f16 bf16; do
  timeout 600 python tools/sweep_check.py --sets ragged,7b,70b_tp8 --out $out | tail -1 >> $O 2>&1
  timeout 600 python tools/sweep_check.py --sets ragged,7b --out $out --kind fgq128 | tail -1 >> $O 2>&1
done
timeout 600 python tools/sweep_check.py --sets ragged,7b --kind int4 --sched cluster --splits 2,3 --ms 1,16,32 | tail -1 >> $O 2>&1
timeout 600 python tools/sweep_check.py --sets ragged,7b --kind int4_128 --sched streamk --splits 3,7 --ms 1,16,32,48 | tail -1 >> $O 2>&1

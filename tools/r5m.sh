mkdir -p gpurun_out
timeout 600 python tools/sweep_check.py --sets ragged > gpurun_out/r5m_sweep_ragged.jsonl 2>&1; echo "rc=$?" >> gpurun_out/r5m_sweep_ragged.jsonl
timeout 600 python tools/sweep_check.py --sets ragged --sched streamk --splits 2,5,9 --ms 1,16,32,48 > gpurun_out/r5m_sweep_ragged_sk.jsonl 2>&1; echo "rc=$?" >> gpurun_out/r5m_sweep_ragged_sk.jsonl
timeout 600 python tools/sweep_check.py --sets ragged --sched cluster --splits 2,3,5,8 --ms 1,16,32 > gpurun_out/r5m_sweep_ragged_csk.jsonl 2>&1; echo "rc=$?" >> gpurun_out/r5m_sweep_ragged_csk.jsonl
for kind in fgq128 fgq32 fp5 int4_128; do
  timeout 600 python tools/sweep_check.py --sets ragged --kind $kind > gpurun_out/r5m_sweep_ragged_$kind.jsonl 2>&1; echo "rc=$?" >> gpurun_out/r5m_sweep_ragged_$kind.jsonl
done

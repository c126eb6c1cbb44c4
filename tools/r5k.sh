mkdir -p gpurun_out
timeout 600 python tools/sweep_check.py --sets 7b,70b,70b_tp8 --sched streamk --splits 0,2,3,5,8,16 --ms 1,16,24,32,48,64 > gpurun_out/r5k_sweep_streamk.jsonl 2>&1; echo "rc=$?" >> gpurun_out/r5k_sweep_streamk.jsonl
timeout 600 python tools/sweep_check.py --sets 7b,70b,70b_tp8 --sched cluster --splits 0,2,3,4,8 --ms 1,16,24,32 > gpurun_out/r5k_sweep_cluster.jsonl 2>&1; echo "rc=$?" >> gpurun_out/r5k_sweep_cluster.jsonl
timeout 600 python tools/sweep_check.py --sets 7b,70b,70b_tp8 --sched pair --splits 0,1,2 --ms 65,128,256,512,1024 > gpurun_out/r5k_sweep_pair.jsonl 2>&1; echo "rc=$?" >> gpurun_out/r5k_sweep_pair.jsonl
timeout 600 python tools/sweep_check.py --sets 7b,70b,70b_tp8 --sched single --splits 0,2,4 --ms 65,128,256,512 > gpurun_out/r5k_sweep_single.jsonl 2>&1; echo "rc=$?" >> gpurun_out/r5k_sweep_single.jsonl

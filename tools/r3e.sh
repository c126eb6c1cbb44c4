mkdir -p gpurun_out
timeout 900 python tools/probe.py --shapes 70b --m 512,2048 --sched pair --split 1,2 > gpurun_out/r3e_probe_force.jsonl 2>&1
timeout 900 python tools/probe.py --shapes 7b,13b --m 512,1024,4096 --sched pair --split 1,2 > gpurun_out/r3e_probe_force_7b.jsonl 2>&1
timeout 900 python tools/probe.py --shapes 70b --m 8192 > gpurun_out/r3e_probe_8192.jsonl 2>&1

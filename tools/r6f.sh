mkdir -p gpurun_out
timeout 900 python tools/container_sweep.py > gpurun_out/r6f_container.jsonl 2>&1; echo "rc=$?" >> gpurun_out/r6f_container.jsonl

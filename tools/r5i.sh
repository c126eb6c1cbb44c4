mkdir -p gpurun_out
timeout 1500 python tools/sweep_check.py > gpurun_out/r5i_sweep.jsonl 2>&1; echo "rc=$?" >> gpurun_out/r5i_sweep.jsonl

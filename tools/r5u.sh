mkdir -p gpurun_out
timeout 1500 python tools/quant_sweep.py > gpurun_out/r5u_quant_sweep.jsonl 2>&1; echo "rc=$?" >> gpurun_out/r5u_quant_sweep.jsonl

mkdir -p gpurun_out
timeout 600 python tools/repro_fgq.py 128 > gpurun_out/r5n_fgq128.jsonl 2>&1

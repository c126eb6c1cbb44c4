#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench_v9.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_v9.log
timeout 600 python bench.py --model llama2-70b --steps 500 > gpurun_out/bench70_v9.log 2>&1
timeout 600 python tools/probe.py --shapes all --m 1,16,64,128,512,2048,8192 > gpurun_out/probe_v9.log 2>&1
python - <<'PY'
import json
for f in ["gpurun_out/bench_v9.log","gpurun_out/bench70_v9.log"]:
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f, d["value"], d["roofline"]["frac"], d["cublas_fp16"]["speedup_vs_cublas"], d["e2e"]["value"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
for l in open("gpurun_out/probe_v9.log"):
    try: d=json.loads(l)
    except: continue
    print(d["n"], d["k"], d["m"], d["plan"]["block_n"], d["plan"]["schedule"], d["plan"]["grid"], d["us_fp6"], d["us_cublas"], d["speedup"], d["TFLOPS"])
PY

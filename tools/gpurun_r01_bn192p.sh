#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
timeout 600 python tools/probe.py --shapes 70b --m 512,2048,8192 > gpurun_out/probe_bn256.log 2>&1
LPQT_LIB=build/variants/lib_bn192.so timeout 600 python tools/probe.py --shapes 70b --m 512,2048,8192 > gpurun_out/probe_bn192.log 2>&1
for f in gpurun_out/probe_bn256.log gpurun_out/probe_bn192.log; do echo $f; python -c "
import json,sys
for l in open('$f'):
    try: d=json.loads(l)
    except: continue
    print(d['n'],d['k'],d['m'],d['us_fp6'],d['us_cublas'],d['speedup'],d['TFLOPS'],d['plan'].get('grid'))
"; done

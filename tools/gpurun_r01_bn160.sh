#!/bin/bash
mkdir -p gpurun_out
timeout 60 env LPQT_LIB=build/variants/lib_bn160.so python tools/abx.py --libs build/variants/lib_bn160.so --shapes 4096x4096 --m 512 --rounds 1 --launches 3 > gpurun_out/bn160_smoke.log 2>&1 || { echo "bn160 smoke failed"; cat gpurun_out/bn160_smoke.log; exit 1; }
timeout 600 python tools/probe.py --shapes 70b --m 512,2048,8192 > gpurun_out/probe_bn192b.log 2>&1
LPQT_LIB=build/variants/lib_bn160.so timeout 600 python tools/probe.py --shapes 70b --m 512,2048,8192 > gpurun_out/probe_bn160.log 2>&1
for f in gpurun_out/probe_bn192b.log gpurun_out/probe_bn160.log; do echo $f; python -c "
import json
for l in open('$f'):
    try: d=json.loads(l)
    except: continue
    print(d['n'],d['k'],d['m'],d['plan']['block_n'],d['plan']['schedule'],d['us_fp6'],d['us_cublas'],d['speedup'],d['TFLOPS'])
"; done

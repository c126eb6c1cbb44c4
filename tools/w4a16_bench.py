"""W4A16 (INT4, fused) vs W6A16 (FP6) vs cuBLAS fp16 launch time (dev tool):
back-to-back launches in a CUDA graph, weights rotated over > 2x L2.
Reports us per launch and the weight stream rate (GB/s of algorithmic bytes).

python tools/w4a16_bench.py [--m 1,16,2048] [--shapes NxK,...]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="12288x4096,22016x4096,57344x8192,8192x28672")
ap.add_argument("--m", default="1,16,2048")
ap.add_argument("--block", type=int, default=0)
a = ap.parse_args()
l2 = torch.cuda.get_device_properties(0).L2_cache_size


def timed(fn, launches):
    fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(launches):
            fn(i)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / launches)
    return sorted(ts)[2]


for shape in a.shapes.split(","):
    n, k = (int(v) for v in shape.split("x"))
    copies = max(2, -(-2 * l2 // (n * k // 2)))
    W = (torch.randn(n, k, device="cuda") * 0.02).half()
    gran = L.Granularity.FGQ if a.block else L.Granularity.CGQ
    q = L.quantize_tensor(W, L.QuantScheme(gran, L.TensorFormat.INT4_ASYM, a.block))
    w4 = [L.Int4Weight.from_quantized(q)]
    w4 += [L.Int4Weight(w4[0].tiles.clone(), w4[0].scales, w4[0].zeros, n, k, a.block) for _ in range(copies - 1)]
    w6 = [L.Fp6Weight.quantize(W, block=a.block) for _ in range(copies)]
    c16 = max(2, -(-2 * l2 // (n * k * 2)))
    wh = [W.clone() for _ in range(c16)]
    del W, q
    for m in (int(v) for v in a.m.split(",")):
        x = torch.randn(m, k, device="cuda").half()
        y = torch.empty(m, n, device="cuda", dtype=torch.float16)
        launches = 20 if m <= 64 else 4
        us = {"int4": timed(lambda i: L.w6a16_linear(x, w4[i % len(w4)], out=y), launches),
              "fp6": timed(lambda i: L.w6a16_linear(x, w6[i % len(w6)], out=y), launches),
              "fp6_sk": timed(lambda i: L.w6a16_linear(x, w6[i % len(w6)], out=y, sched="streamk"), launches),
              "fp16": timed(lambda i: torch.matmul(x, wh[i % len(wh)].t(), out=y), launches)}
        print(json.dumps({"plan_fp6": L.plan(m, n, k), "plan_fp6_sk": L.plan(m, n, k, sched="streamk")}))
        gbs = {"int4": w4[0].stream_bytes() / us["int4"] / 1e3, "fp6": w6[0].stream_bytes() / us["fp6"] / 1e3,
               "fp16": n * k * 2 / us["fp16"] / 1e3}
        print(json.dumps({"n": n, "k": k, "m": m, "block": a.block,
                          "us": {kk: round(v, 2) for kk, v in us.items()},
                          "weight_GBps": {kk: round(v) for kk, v in gbs.items()},
                          "int4_vs_fp16": round(us["fp16"] / us["int4"], 2),
                          "int4_vs_fp6": round(us["fp6"] / us["int4"], 2)}), flush=True)
    del w4, w6, wh
    torch.cuda.empty_cache()

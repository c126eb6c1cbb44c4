"""Native 5-bit FP5 tiles (0.625 B / weight) vs FP5 widened to FP6 tiles
(0.75 B / weight) vs FP6, decode batches (dev tool).  Single launches
replayed from a CUDA graph, L2 flushed between replays; GB/s are each
format's own algorithmic bytes.

python tools/fp5_bench.py [--m 1,8,16] [--shapes 70b|7b]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402
from paper_2312_08583_b200.linear import prepack  # noqa: E402
from tools.probe import SHAPES, time_fn  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", default="1,8,16")
ap.add_argument("--shapes", default="70b")
a = ap.parse_args()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for n, k in SHAPES[a.shapes]:
    W = (torch.randn(n, k, device="cuda") * 0.02).half()
    q5 = L.quantize_tensor(W, L.QuantScheme(L.Granularity.CGQ, L.TensorFormat.FP5_E3M1), bias_shift=True)
    w5 = L.Fp6Weight.from_quantized(q5)
    s4 = L.quantizer.device_planes(q5)
    w5w = L.Fp6Weight(prepack(s4[0], s4[1], n, k, "fp5"), s4[2], n, k, static=True)
    w6 = L.Fp6Weight.quantize(W)
    del W
    for m in (int(v) for v in a.m.split(",")):
        x = torch.randn(m, k, device="cuda").half()
        y = torch.empty(m, n, device="cuda", dtype=torch.float16)
        res = {}
        for name, w in (("fp5_native", w5), ("fp5_widened", w5w), ("fp6", w6)):
            t = time_fn(lambda: L.w6a16_linear(x, w, out=y), flush=flush)
            res[name] = {"us": round(t * 1e6, 2),
                         "GBps": round((w.stream_bytes() + 2 * m * k + 2 * m * n) / t / 1e9, 1)}
        print(json.dumps({"n": n, "k": k, "m": m, **res,
                          "native_over_widened": round(res["fp5_native"]["us"] / res["fp5_widened"]["us"], 3)}),
              flush=True)

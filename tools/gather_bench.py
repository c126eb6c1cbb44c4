"""Fused GEMM + all-gather epilogue cost on one GPU (dev tool): the 70B TP=8
shard shapes at decode, plain launch vs `lpqt_w6a16_linear_gather` with one
peer (the own buffer: direct stores + system fence + counter + flag barrier),
back-to-back launches in a CUDA graph, weights rotated over > 2x L2.

python tools/gather_bench.py [--m 16]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402
from paper_2312_08583_b200 import _lib, tp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="1280x8192,8192x1024,7168x8192,8192x3584")
ap.add_argument("--m", type=int, default=16)
a = ap.parse_args()
l2 = torch.cuda.get_device_properties(0).L2_cache_size
for shape in a.shapes.split(","):
    n, k = (int(v) for v in shape.split("x"))
    copies = max(2, -(-3 * l2 // (n * k * 3 // 4)))
    W = (torch.randn(n, k, device="cuda") * 0.02).half()
    ws = [L.Fp6Weight.quantize(W) for _ in range(copies)]
    x = torch.randn(a.m, k, device="cuda").half()
    y = torch.empty(a.m, n, device="cuda", dtype=torch.float16)
    flags = torch.zeros(_lib.MAX_PEERS, dtype=torch.int32, device="cuda")
    done = torch.zeros(1, dtype=torch.int32, device="cuda")
    ep = [0]

    def plain(i):
        L.w6a16_linear(x, ws[i % copies], out=y)

    def fused(i):
        ep[0] += 1
        tp.gather_linear(ws[i % copies], x, k, a.m, [y.data_ptr()], [flags.data_ptr()], 0, ep[0], done, _lib.F16,
                         "mn", n, 0)

    res = {}
    for name, fn in (("plain", plain), ("gather1", fused)):
        for i in range(copies):
            fn(i)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(40):
                fn(i)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / 40)
        res[name] = round(sorted(ts)[2], 2)
    print(json.dumps({"n": n, "k": k, "m": a.m, "us": res}), flush=True)

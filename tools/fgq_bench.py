"""FGQ (block scales) vs CGQ W6A16 launch time on the same shapes (dev tool):
back-to-back PDL launches in a CUDA graph, weights rotated over > 2x L2.

python tools/fgq_bench.py [--block 128] [--m 1,16,2048]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="12288x4096,22016x4096,57344x8192,8192x28672")
ap.add_argument("--m", default="1,16,2048")
ap.add_argument("--block", type=int, default=128)
a = ap.parse_args()
l2 = torch.cuda.get_device_properties(0).L2_cache_size
for shape in a.shapes.split(","):
    n, k = (int(v) for v in shape.split("x"))
    copies = max(2, -(-2 * l2 // (n * k * 3 // 4)))
    W = (torch.randn(n, k, device="cuda") * 0.02).half()
    variants = {"cgq": [L.Fp6Weight.quantize(W) for _ in range(copies)],
                f"fgq{a.block}": [L.Fp6Weight.quantize(W, block=a.block) for _ in range(copies)]}
    del W
    for m in (int(v) for v in a.m.split(",")):
        x = torch.randn(m, k, device="cuda").half()
        y = torch.empty(m, n, device="cuda", dtype=torch.float16)
        res = {}
        for name, ws in variants.items():
            launches = 20 if m <= 64 else 4
            for w in ws:
                L.w6a16_linear(x, w, out=y)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(launches):
                    L.w6a16_linear(x, ws[i % copies], out=y)
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3 / launches)
            res[name] = round(sorted(ts)[2], 2)
        print(json.dumps({"n": n, "k": k, "m": m, "us": res}), flush=True)
    del variants
    torch.cuda.empty_cache()

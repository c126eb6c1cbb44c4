"""A/B timing of one W6A16 shape the way bench.py runs it (dev tool):
back-to-back launches captured in a CUDA graph, weights rotated over enough
distinct copies to exceed 2x L2 (every launch reads cold weights, no dirty
L2 from a write-flush), PDL between launches.  Prints us/launch and GB/s.

LPQT_LIB=build/variants/lib_x.so python tools/abbench.py --shapes 8192x28672,22016x4096 --m 16
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="8192x28672,22016x4096,4096x4096,57344x8192")
ap.add_argument("--m", default="16")
ap.add_argument("--launches", type=int, default=40)
ap.add_argument("--split", type=int, default=0)
ap.add_argument("--sched", default="auto")
a = ap.parse_args()
l2 = torch.cuda.get_device_properties(0).L2_cache_size
for shape in a.shapes.split(","):
    n, k = (int(v) for v in shape.split("x"))
    wbytes = n * k * 3 // 4
    copies = max(2, -(-3 * l2 // wbytes))
    g = torch.Generator(device="cuda").manual_seed(0)
    W0 = (torch.randn(n, k, device="cuda", generator=g) * 0.02).half()
    w0 = L.Fp6Weight.quantize(W0)
    del W0
    ws = [w0] + [L.Fp6Weight(w0.tiles.clone(), w0.scales.clone(), n, k, static=True) for _ in range(copies - 1)]
    torch.cuda.synchronize()
    for m in (int(v) for v in a.m.split(",")):
        x = torch.randn(m, k, device="cuda").half()
        y = torch.empty(m, n, device="cuda", dtype=torch.float16)
        for w in ws:
            L.w6a16_linear(x, w, out=y, split_k=a.split, sched=a.sched)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for i in range(a.launches):
                L.w6a16_linear(x, ws[i % copies], out=y, split_k=a.split, sched=a.sched)
        graph.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            graph.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / a.launches)
        t = sorted(ts)[len(ts) // 2]
        byt = w0.stream_bytes() + 2 * m * k + 2 * m * n
        print(json.dumps({"lib": os.path.basename(os.environ.get("LPQT_LIB", "default")) + ":" + a.sched,
                          "n": n, "k": k, "m": m,
                          "copies": copies, "us": round(t, 2), "GBps": round(byt / t / 1e3, 1),
                          "plan": L.plan(m, n, k, a.split, sched=a.sched)}), flush=True)
    del ws, w0
    torch.cuda.empty_cache()

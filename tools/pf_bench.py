"""Cross-launch L2 prefetch A/B on a decode chain (dev tool).

The LLaMA-2 7B (or 70B) block's four linears run back to back as PDL
launches in one CUDA graph per weight copy (copies rotated, > 2x L2); with
prefetch each launch names the next launch's weight (the last one the next
copy's first layer).  Prints us/step and GB/s per prefetch depth.

python tools/pf_bench.py [--model 7b|70b] [--m 16] [--depths 0,32768,65536]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402

SHAPES = {"7b": [(12288, 4096), (4096, 4096), (22016, 4096), (4096, 11008)],
          "70b": [(10240, 8192), (8192, 8192), (57344, 8192), (8192, 28672)]}
ap = argparse.ArgumentParser()
ap.add_argument("--model", default="7b")
ap.add_argument("--m", type=int, default=16)
ap.add_argument("--depths", default="-1,16384,32768,65536,131072,262144")
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--rounds", type=int, default=5)
ap.add_argument("--plans", default="", help="per-layer sched:split overrides, e.g. cluster:2,auto:0,streamk:0,auto:0")
a = ap.parse_args()
shapes = SHAPES[a.model]
l2 = torch.cuda.get_device_properties(0).L2_cache_size
set_bytes = sum(n * k * 3 // 4 for n, k in shapes)
copies = max(2, -(-2 * l2 // set_bytes))
g = torch.Generator(device="cuda").manual_seed(0)
base = []
for n, k in shapes:
    W = (torch.randn(n, k, device="cuda", generator=g) * 0.02).half()
    base.append(L.Fp6Weight.quantize(W))
    del W
sets = [base] + [[L.Fp6Weight(w.tiles.clone(), w.scales.clone(), w.n, w.k, static=True) for w in base]
                 for _ in range(copies - 1)]
m = a.m
xs = [torch.randn(m, k, device="cuda").half() for _, k in shapes]
ys = [torch.empty(m, n, device="cuda", dtype=torch.float16) for n, _ in shapes]


plans = [(p.split(":")[0], int(p.split(":")[1])) for p in a.plans.split(",")] if a.plans else [("auto", 0)] * len(shapes)


def step(c, depth):
    for i, w in enumerate(sets[c]):
        nxt = None
        if depth >= 0:
            nxt = sets[c][i + 1] if i + 1 < len(shapes) else sets[(c + 1) % copies][0]
        L.w6a16_linear(xs[i], w, out=ys[i], prefetch=nxt, prefetch_bytes=max(depth, 0), sched=plans[i][0],
                       split_k=plans[i][1])


depths = [int(v) for v in a.depths.split(",")]
graphs = {}
for d in depths:
    for c in range(copies):
        step(c, d)
    torch.cuda.synchronize()
    gs = []
    for c in range(copies):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            step(c, d)
        gs.append(gr)
    graphs[d] = gs
times = {d: [] for d in depths}
for r in range(a.rounds):
    for d in depths:
        for c in range(copies):
            graphs[d][c].replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in range(a.steps):
            graphs[d][s % copies].replay()
        e1.record()
        torch.cuda.synchronize()
        times[d].append(e0.elapsed_time(e1) * 1e3 / a.steps)
byt = sum(w.stream_bytes() for w in base) + sum(2 * m * k + 2 * m * n for n, k in shapes)
for d in depths:
    t = sorted(times[d])[len(times[d]) // 2]
    print(json.dumps({"model": a.model, "m": m, "plans": a.plans or "auto", "prefetch_bytes_per_cta": d, "us_per_step": round(t, 2),
                      "min": round(min(times[d]), 2), "GBps": round(byt / t / 1e3, 1)}), flush=True)

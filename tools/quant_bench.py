"""Time the GPU quantizers (dev tool): Fp6Weight.quantize (scales + encode
straight into tiles) and quantize_tensor (scales + encode into canonical
planes) + prepack, on LLaMA-2 shapes, f16 and bf16 input.

python tools/quant_bench.py [--shapes 57344x8192,8192x28672]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="57344x8192,8192x28672,12288x4096,4096x4096")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
CGQ = L.QuantScheme(L.Granularity.CGQ, L.TensorFormat.FP6_E3M2)


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return sorted(ts)[len(ts) // 2]


for shape in a.shapes.split(","):
    n, k = (int(v) for v in shape.split("x"))
    for dt in (torch.float16, torch.bfloat16):
        W = (torch.randn(n, k, device="cuda") * 0.02).to(dt)
        t_tiles = timed(lambda: L.Fp6Weight.quantize(W), a.reps)

        def planes():
            q = L.quantize_tensor(W, CGQ, bias_shift=True)
            return L.Fp6Weight.from_planes(q.payload.seg4, q.payload.seg_tail, q.scales, n, k, q.folded_scales)
        t_planes = timed(planes, a.reps)
        # algorithmic bytes of the tiles path: read W twice (scales pass, encode pass) + write 0.75 B/weight
        byt = n * k * (2 * W.element_size() + 0.75)
        print(json.dumps({"n": n, "k": k, "dtype": str(dt).split(".")[-1], "tiles_us": round(t_tiles, 1),
                          "tiles_GBps": round(byt / t_tiles / 1e3, 1), "planes_plus_prepack_us": round(t_planes, 1),
                          "Mweights_per_ms": round(n * k / t_tiles / 1e3, 1)}), flush=True)
        del W
    torch.cuda.empty_cache()

"""Stress the stream-K / cluster reductions for bit-determinism (dev tool).
Runs the same launch many times (optionally alternating with a prefetch
hint, which perturbs timing) and counts results that differ from the first.

LPQT_LIB=... python tools/determinism_stress.py --shape 4096x11008 --m 1 --reps 300
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096x11008")
ap.add_argument("--m", type=int, default=1)
ap.add_argument("--reps", type=int, default=300)
ap.add_argument("--sched", default="auto")
a = ap.parse_args()
n, k = (int(v) for v in a.shape.split("x"))
g = torch.Generator(device="cuda").manual_seed(3)
w = L.Fp6Weight.quantize((torch.randn(n, k, device="cuda", generator=g) * 0.02).half())
w2 = L.Fp6Weight.quantize((torch.randn(640, 256, device="cuda", generator=g) * 0.02).half())
x = torch.randn(a.m, k, device="cuda", generator=g).half()
ref = L.w6a16_linear(x, w, out_dtype=torch.float32, sched=a.sched)
bad = {"plain": 0, "prefetch": 0}
maxdiff = 0.0
for r in range(a.reps):
    for mode in ("plain", "prefetch"):
        y = L.w6a16_linear(x, w, out_dtype=torch.float32, sched=a.sched, prefetch=w2 if mode == "prefetch" else None)
        if not torch.equal(y, ref):
            bad[mode] += 1
            d = (y - ref).abs()
            maxdiff = max(maxdiff, float(d.max()))
            if bad[mode] <= 2:
                idx = torch.nonzero(d).tolist()[:4]
                print(mode, r, "rows differ:", sorted({i[1] // 128 for i in torch.nonzero(d).tolist()})[:10], idx)
print({"shape": a.shape, "m": a.m, "plan": L.plan(a.m, n, k, 0, sched=a.sched), "bad": bad, "maxdiff": maxdiff,
       "lib": os.environ.get("LPQT_LIB", "default")})

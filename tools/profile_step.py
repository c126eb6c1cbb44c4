"""Run the bench step's four W6A16 GEMMs once each, eagerly (target for
`ncu --set full -k regex:w6a16 -c 4`): the per-launch DRAM traffic of the
step's kernels, for bench.py's roofline.traffic (profiles/ncu_traffic.json).

python tools/profile_step.py [--model llama2-7b] [--m 16]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402
from bench import LAYERS_7B, LAYERS_70B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama2-7b")
ap.add_argument("--m", type=int, default=16)
a = ap.parse_args()
layers = LAYERS_7B if a.model == "llama2-7b" else LAYERS_70B
ws, xs, ys = [], [], []
for _, n, k in layers:
    W = (torch.randn(n, k, device="cuda") * 0.02).half()
    ws.append(L.Fp6Weight.quantize(W))
    del W
    xs.append(torch.randn(a.m, k, device="cuda").half())
    ys.append(torch.empty(a.m, n, device="cuda", dtype=torch.float16))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for rep in range(2):   # rep 0 warms up; ncu -s skips its launches
    for i in range(len(layers)):
        flush.sum()
        L.w6a16_linear(xs[i], ws[i], out=ys[i])
torch.cuda.synchronize()
print("plans", [L.plan(a.m, n, k) for _, n, k in layers])

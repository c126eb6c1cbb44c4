"""Run one W6A16 GEMM shape a few times eagerly (target for `ncu -k regex:w6a16`).

python tools/profile_one.py --n 22016 --k 4096 --m 16 [--iters 5] [--split 0]
"""

import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=22016)
ap.add_argument("--k", type=int, default=4096)
ap.add_argument("--m", type=int, default=16)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--split", type=int, default=0)
a = ap.parse_args()
W = (torch.randn(a.n, a.k, device="cuda") * 0.02).half()
w = L.Fp6Weight.quantize(W)
x = torch.randn(a.m, a.k, device="cuda").half()
y = torch.empty(a.m, a.n, device="cuda", dtype=torch.float16)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(a.iters):
    flush.zero_()
    L.w6a16_linear(x, w, out=y, split_k=a.split)
torch.cuda.synchronize()
print("plan", L.plan(a.m, a.n, a.k, a.split), "bytes", w.stream_bytes())

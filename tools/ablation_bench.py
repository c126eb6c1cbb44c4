"""The paper's Bias-Shift ablation on B200 (presets
PAPER.md:487-497): the FP6 decode GEMM with the hardware e3m2 rebuild (product
path), the software bias-shift rebuild and the naive two-step rebuild (both x
per-weight binary16 scale), at the paper's batch 8, next to cuBLAS fp16.
Single launches replayed from a CUDA graph, L2 flushed between replays.

python tools/ablation_bench.py [--m 8] [--shapes paper|70b]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402
from tools.probe import time_fn  # noqa: E402

PAPER = [(5504, 2048), (2048, 5504), (13824, 5120), (5120, 13824), (22016, 8192), (8192, 22016)]
B70 = [(10240, 8192), (8192, 8192), (57344, 8192), (8192, 28672)]
ap = argparse.ArgumentParser()
ap.add_argument("--m", default="8")
ap.add_argument("--shapes", default="paper")
a = ap.parse_args()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for n, k in (PAPER if a.shapes == "paper" else B70):
    W = (torch.randn(n, k, device="cuda") * 0.02).half()
    w = L.Fp6Weight.quantize(W)
    for m in (int(v) for v in a.m.split(",")):
        x = torch.randn(m, k, device="cuda").half()
        y = torch.empty(m, n, device="cuda", dtype=torch.float16)
        us = {}
        for rb in ("cvt", "bias_shift", "naive"):
            us[rb] = round(time_fn(lambda: L.w6a16_linear(x, w, out=y, rebuild=rb), flush=flush) * 1e6, 2)
        us["cublas_fp16"] = round(time_fn(lambda: torch.matmul(x, W.t()), flush=flush) * 1e6, 2)
        wbytes = w.stream_bytes() + 2 * m * k + 2 * m * n
        print(json.dumps({"n": n, "k": k, "m": m, "us": us,
                          "naive_over_bias_shift": round(us["naive"] / us["bias_shift"], 3),
                          "bias_shift_over_cvt": round(us["bias_shift"] / us["cvt"], 3),
                          "GBps": {r: round(wbytes / (us[r] * 1e-6) / 1e9, 1) for r in ("cvt", "bias_shift", "naive")},
                          "plan": L.plan(m, n, k)}), flush=True)

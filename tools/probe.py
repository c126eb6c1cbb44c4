"""Quick kernel timing probe (dev tool): W6A16 vs cuBLAS fp16 on a few shapes.

python tools/probe.py [--shapes 7b|70b|all] [--m 1,16]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402

SHAPES = {
    "7b": [(12288, 4096), (4096, 4096), (22016, 4096), (4096, 11008)],
    "70b": [(10240, 8192), (8192, 8192), (57344, 8192), (8192, 28672)],
    # BASELINE configs[2]: LLaMA-2-13B and StarCoder-15B (MQA, MLP 24576)
    "13b": [(15360, 5120), (5120, 5120), (27648, 5120), (5120, 13824)],
    "sc15b": [(6400, 6144), (6144, 6144), (24576, 6144), (6144, 24576)],
}
# BASELINE configs[3]: the 70B layers column-sharded over P GPUs (one rank's shard)
for _p in (2, 4, 8):
    SHAPES[f"70b_tp{_p}"] = [(n // _p, k) for n, k in SHAPES["70b"]]


def time_fn(fn, iters=50, warm=5, flush=None):
    """Median device time of one call, replayed from a CUDA graph (no host
    launch overhead inside the events), L2 flushed between replays."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    evs = []
    for _ in range(iters):
        if flush is not None:
            flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    return ts[len(ts) // 2] * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="all")
    ap.add_argument("--m", default="1,16")
    ap.add_argument("--split", default="0", help="comma list of split_k values (0 = automatic plan)")
    ap.add_argument("--sched", default="auto", help="auto / pair / single / streamk / cluster")
    args = ap.parse_args()
    shapes = SHAPES["7b"] + SHAPES["70b"] if args.shapes == "all" else sum((SHAPES[s] for s in args.shapes.split(",")), [])
    splits = [int(v) for v in args.split.split(",")]
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for n, k in shapes:
        W = (torch.randn(n, k, device="cuda") * 0.02).half()
        lin = L.Fp6Linear.from_dense(W)
        for m, split in ((int(v), sp) for v in args.m.split(",") for sp in splits):
            x = torch.randn(m, k, device="cuda").half()
            y = torch.empty(m, n, device="cuda", dtype=torch.float16)
            t6 = time_fn(lambda: L.w6a16_linear(x, lin.weight, out=y, split_k=split, sched=args.sched), flush=flush)
            t16 = time_fn(lambda: torch.matmul(x, W.t()), flush=flush)
            ref = (x.float() @ W.float().t())
            err = float((y.float() - ref).abs().max() / ref.abs().max())
            wbytes = lin.weight.stream_bytes() + 2 * m * k + 2 * m * n
            print(json.dumps({"n": n, "k": k, "m": m, "split_k": split, "plan": L.plan(m, n, k, split, sched=args.sched),
                              "us_fp6": round(t6 * 1e6, 2), "us_cublas": round(t16 * 1e6, 2),
                              "speedup": round(t16 / t6, 3), "GBps": round(wbytes / t6 / 1e9, 1),
                              "TFLOPS": round(2 * m * n * k / t6 / 1e12, 2), "err_vs_fp16W": err}), flush=True)


if __name__ == "__main__":
    main()

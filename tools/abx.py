"""Interleaved A/B of several liblpqt_b200 builds in ONE process (dev tool).

Each library is loaded with its own ctypes handle; for every shape the same
weights / activations are timed under every library in turn, ROUNDS times
interleaved (A B C A B C ...), as back-to-back PDL launches in a CUDA graph
with weights rotated over > 3x L2.  Prints the median us/launch per library.

python tools/abx.py --libs paper_2312_08583_b200/liblpqt_b200.so,build/variants/lib_prev.so \
    --shapes 57344x8192,4096x4096 --m 16 [--flags 0,2]
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L  # noqa: E402
from paper_2312_08583_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--libs", required=True)
ap.add_argument("--flags", default="", help="per-lib extra flags (2 = stream-K, 4 = cluster)")
ap.add_argument("--splits", default="", help="per-lib split_k")
ap.add_argument("--shapes", default="57344x8192,8192x28672,22016x4096,12288x4096,4096x4096")
ap.add_argument("--m", default="16")
ap.add_argument("--launches", type=int, default=30)
ap.add_argument("--rounds", type=int, default=5)
a = ap.parse_args()

paths = a.libs.split(",")
flags = [int(v) for v in a.flags.split(",")] if a.flags else [0] * len(paths)
splits = [int(v) for v in a.splits.split(",")] if a.splits else [0] * len(paths)
libs = []
for p in paths:
    lib = ctypes.CDLL(os.path.abspath(p))
    f = lib.lpqt_w6a16_linear_ex
    f.restype = ctypes.c_int
    f.argtypes = _lib.SIGNATURES["lpqt_w6a16_linear_ex"][1]
    w = lib.lpqt_w6a16_workspace_bytes
    w.restype = ctypes.c_int64
    w.argtypes = _lib.SIGNATURES["lpqt_w6a16_workspace_bytes"][1]
    libs.append(lib)
l2 = torch.cuda.get_device_properties(0).L2_cache_size
ws_buf = torch.zeros(160 << 20, dtype=torch.uint8, device="cuda")

for shape in a.shapes.split(","):
    n, k = (int(v) for v in shape.split("x"))
    copies = max(2, -(-3 * l2 // (n * k * 3 // 4)))
    W0 = (torch.randn(n, k, device="cuda") * 0.02).half()
    w0 = L.Fp6Weight.quantize(W0)
    del W0
    tiles = [w0.tiles] + [w0.tiles.clone() for _ in range(copies - 1)]
    for m in (int(v) for v in a.m.split(",")):
        x = torch.randn(m, k, device="cuda").half()
        y = torch.empty(m, n, device="cuda", dtype=torch.float16)
        graphs = []
        for li, lib in enumerate(libs):
            # (the query knows no schedule flags: a forced pair plan needs far less
            # than the single-SM split it sizes; the launch itself checks the size)
            need = lib.lpqt_w6a16_workspace_bytes(m, n, k, splits[li])
            assert need <= ws_buf.numel() or flags[li] & 16, need

            def call(t, lib=lib, li=li):
                st = lib.lpqt_w6a16_linear_ex(t.data_ptr(), w0.scales.data_ptr(), x.data_ptr(), k, m, n, k,
                                              y.data_ptr(), _lib.F16, _lib.Y_MN, n, splits[li], ws_buf.data_ptr(),
                                              ws_buf.numel(), 1 | flags[li], torch.cuda.current_stream().cuda_stream)
                assert st == 0, st
            for t in tiles:
                call(t)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(a.launches):
                    call(tiles[i % copies])
            g.replay()
            torch.cuda.synchronize()
            graphs.append(g)
        times = [[] for _ in libs]
        for _ in range(a.rounds):
            for li, g in enumerate(graphs):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                times[li].append(e0.elapsed_time(e1) * 1e3 / a.launches)
        byt = w0.stream_bytes() + 2 * m * k + 2 * m * n
        print(json.dumps({"n": n, "k": k, "m": m,
                          "us": {os.path.basename(p) + (f"/f{flags[i]}s{splits[i]}" if a.flags or a.splits else ""):
                                 [round(statistics.median(times[i]), 2), round(min(times[i]), 2),
                                  round(max(times[i]), 2)] for i, p in enumerate(paths)},
                          "GBps_best": round(byt / min(min(t) for t in times) / 1e3, 1)}), flush=True)
        del graphs
    del tiles, w0
    torch.cuda.empty_cache()

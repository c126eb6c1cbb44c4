"""Per-CTA timeline of back-to-back W6A16 launches (PDL chain) with the
LPQT_TRACE library (dev tool).  Launches a chain of the given shapes (like one
bench step), eagerly, and prints per launch: first CTA entry, X-wait release,
median/max CTA exit, all relative to the first launch's first entry (us).

LPQT_LIB=build/variants/lib_trace.so python tools/chain_trace.py --shapes 12288x4096,4096x4096,22016x4096,4096x11008 --m 16
"""
import argparse, ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L
from paper_2312_08583_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="12288x4096,4096x4096,22016x4096,4096x11008")
ap.add_argument("--m", type=int, default=16)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--sched", default="auto")
ap.add_argument("--split", type=int, default=0)
ap.add_argument("--graph", action="store_true", help="replay the chain from a CUDA graph (PDL edges back to back)")
a = ap.parse_args()
shapes = [tuple(int(v) for v in s.split("x")) for s in a.shapes.split(",")]
ws, xs, ys = [], [], []
for n, k in shapes:
    W = (torch.randn(n, k, device="cuda") * 0.02).half()
    ws.append(L.Fp6Weight.quantize(W))
    xs.append(torch.randn(a.m, k, device="cuda").half())
    ys.append(torch.empty(a.m, n, device="cuda", dtype=torch.float16))
lib = _lib.load()
lib.lpqt_trace_dump_all.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
SLOTS, LEN = 16, 256 * 24
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
if a.graph:
    for i in range(len(shapes)):  # warm-up (workspace, attributes) before capture
        L.w6a16_linear(xs[i], ws[i], out=ys[i], sched=a.sched, split_k=a.split)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(len(shapes)):
            L.w6a16_linear(xs[i], ws[i], out=ys[i], sched=a.sched, split_k=a.split)
for rep in range(a.reps):
    flush.sum()  # read-only L2 flush (clean lines)
    torch.cuda.synchronize()
    if a.graph:
        g.replay()
    else:
        for i in range(len(shapes)):
            L.w6a16_linear(xs[i], ws[i], out=ys[i], sched=a.sched, split_k=a.split)
    torch.cuda.synchronize()
buf = (ctypes.c_longlong * (SLOTS * LEN))()
n = ctypes.c_int(0)
lib.lpqt_trace_dump_all(buf, ctypes.byref(n))
t = np.frombuffer(buf, dtype=np.int64).reshape(SLOTS, LEN)
last = [(n.value - len(shapes) + j) % SLOTS for j in range(len(shapes))]
recs = []
for j, slot in enumerate(last):
    nn, kk = shapes[j]
    g = L.plan(a.m, nn, kk, a.split, sched=a.sched)["grid"]
    c = t[slot, : 256 * 24].reshape(256, 24)[:g].astype(np.float64)
    recs.append(c)
t0 = recs[0][:, 0].min()
print("times in us from the chain's first CTA entry")
print(f"{'shape':>12} {'entry0':>7} {'entryMx':>7} {'xwait':>7} {'1stdata':>7} {'prodWmed':>8} {'mmaMed':>7} {'exitMed':>7} {'exitMax':>7}")
for j, c in enumerate(recs):
    r = lambda col: (c[:, col] - t0) / 1e3
    print(f"{'%dx%d' % shapes[j]:>12} {r(0).min():7.2f} {r(0).max():7.2f} {np.median(r(13)):7.2f} {np.median(r(12)):7.2f} "
          f"{np.median(r(2)):8.2f} {np.median(r(4)):7.2f} {np.median(r(6)):7.2f} {r(6).max():7.2f}")
cols = [0, 1, 12, 13, 14, 2, 3, 16, 4, 15, 17, 18, 8, 11, 5, 6]
names = ["entry", "setup", "dq1st", "xok", "mma1x", "prodW", "dq0dn", "dq1dn", "mmadn", "mma1dn", "e_clw", "e_pdl",
         "e_dfull", "e_fix", "epidn", "exit"]
for j, c in enumerate(recs):
    rel = np.where(c[:, cols] > 0, (c[:, cols] - t0) / 1e3, np.nan)
    order = np.argsort(rel[:, -1])
    print(f"--- {shapes[j]}: fastest 2 / slowest 4 CTAs")
    print("  cta | " + " ".join(f"{nm:>7}" for nm in names))
    for ci in list(order[:2]) + list(order[-4:]):
        print(f" {ci:4d} | " + " ".join(f"{v:7.2f}" for v in rel[ci]))

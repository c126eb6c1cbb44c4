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
ap.add_argument("--pf", type=int, default=-1, help="prefetch the next launch's weights (bytes per CTA; -1 = off)")
ap.add_argument("--graph", action="store_true", help="replay the chain from a CUDA graph (PDL edges back to back)")
a = ap.parse_args()
shapes = [tuple(int(v) for v in s.split("x")) for s in a.shapes.split(",")]
ws, xs, ys = [], [], []


def pfk(i):
    if a.pf < 0:
        return {}
    return {"prefetch": ws[(i + 1) % len(ws)], "prefetch_bytes": a.pf}



for n, k in shapes:
    W = (torch.randn(n, k, device="cuda") * 0.02).half()
    ws.append(L.Fp6Weight.quantize(W))
    xs.append(torch.randn(a.m, k, device="cuda").half())
    ys.append(torch.empty(a.m, n, device="cuda", dtype=torch.float16))
lib = _lib.load()
lib.lpqt_trace_dump_all.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
SLOTS, LEN = 16, 256 * 32
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
if a.graph:
    for i in range(len(shapes)):  # warm-up (workspace, attributes) before capture
        L.w6a16_linear(xs[i], ws[i], out=ys[i], sched=a.sched, split_k=a.split)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(len(shapes)):
            L.w6a16_linear(xs[i], ws[i], out=ys[i], sched=a.sched, split_k=a.split, **pfk(i))
for rep in range(a.reps):
    flush.sum()  # read-only L2 flush (clean lines)
    torch.cuda.synchronize()
    if a.graph:
        g.replay()
    else:
        for i in range(len(shapes)):
            L.w6a16_linear(xs[i], ws[i], out=ys[i], sched=a.sched, split_k=a.split, **pfk(i))
    torch.cuda.synchronize()
buf = (ctypes.c_longlong * (SLOTS * LEN))()
n = ctypes.c_int(0)
lib.lpqt_trace_dump_all(buf, ctypes.byref(n))
t = np.frombuffer(buf, dtype=np.int64).reshape(SLOTS, LEN)
last = [(n.value - len(shapes) + j) % SLOTS for j in range(len(shapes))]
recs = []
G0 = [None]


def gbase_off(gb):  # all launches on one axis: offsets from the first launch's base
    if G0[0] is None:
        G0[0] = gb
    return float(gb - G0[0])


for j, slot in enumerate(last):
    nn, kk = shapes[j]
    g = L.plan(a.m, nn, kk, a.split, sched=a.sched)["grid"]
    ri = t[slot, : 256 * 32].reshape(256, 32)[:g]
    # stamps are %clock64; slots 30/31 hold %globaltimer at entry / exit.
    # Offsets are taken in int64 first: ns timestamps (~1.8e18) do not fit a
    # float64 mantissa (256 ns quantisation).
    gbase = ri[:, 30].min()
    raw = np.zeros(ri.shape)
    raw[:, :30] = np.where(ri[:, :30] != 0, (ri[:, :30] - ri[:, 0:1]).astype(np.float64), -1.0)
    raw[:, 30:32] = (ri[:, 30:32] - gbase).astype(np.float64)
    ck0, ck6, gt0, gt6 = np.zeros((g, 1)), raw[:, 6:7], raw[:, 30:31], raw[:, 31:32]
    raw[:, 0] = 0.0
    ns_per_ck = (gt6 - gt0) / np.maximum(ck6 - ck0, 1)
    c = np.where(raw[:, :30] >= 0, gt0 + (raw[:, :30] - ck0) * ns_per_ck + gbase_off(gbase), np.nan)
    recs.append(c)
    if os.environ.get("TRACE_RAW"):
        print("raw", shapes[j], raw[:3][:, [0, 19, 20, 1, 12, 6, 30, 31]].astype(np.int64).tolist(), ns_per_ck[:3].ravel())
t0 = np.nanmin(recs[0][:, 0])
print("times in us from the chain's first CTA entry")
print(f"{'shape':>12} {'entry0':>7} {'entryMx':>7} {'xwait':>7} {'1stdata':>7} {'prodWmed':>8} {'mmaMed':>7} {'exitMed':>7} {'exitMax':>7}")
for j, c in enumerate(recs):
    r = lambda col: (c[:, col] - t0) / 1e3
    print(f"{'%dx%d' % shapes[j]:>12} {np.nanmin(r(0)):7.2f} {np.nanmax(r(0)):7.2f} {np.nanmedian(r(13)):7.2f} "
          f"{np.nanmedian(r(12)):7.2f} {np.nanmedian(r(2)):8.2f} {np.nanmedian(r(4)):7.2f} {np.nanmedian(r(6)):7.2f} "
          f"{np.nanmax(r(6)):7.2f}")
cols = [0, 19, 20, 21, 22, 1, 12, 13, 14, 2, 3, 16, 4, 15, 17, 18, 8, 9, 10, 23, 26, 27, 24, 25, 11, 5, 6]
names = ["entry", "binit", "w1iss", "talloc", "dqreg", "setup", "dq1st", "xok", "mma1x", "prodW", "dq0dn", "dq1dn", "mmadn", "mma1dn", "e_clw", "e_pdl",
         "e_dfull", "e_pub", "e_atom", "e_gath", "e_own", "e_add", "e_sum", "e_yend", "e_fix", "epidn", "exit"]
for j, c in enumerate(recs):
    rel = (c[:, cols] - t0) / 1e3
    order = np.argsort(np.nan_to_num(rel[:, -1]))
    print(f"--- {shapes[j]}: fastest 2 / slowest 4 CTAs")
    print("  cta | " + " ".join(f"{nm:>7}" for nm in names))
    for ci in list(order[:2]) + list(order[-4:]):
        print(f" {ci:4d} | " + " ".join(f"{v:7.2f}" for v in rel[ci]))

"""Run one GEMM with the LPQT_TRACE library and print the per-CTA timeline
(%globaltimer stamps) plus the CTA-0 event table (clock64).

LPQT_LIB=build/variants/lib_trace.so python tools/trace_run.py --n 22016 --k 4096 --m 16"""
import argparse, ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_08583_b200 as L
from paper_2312_08583_b200 import _lib
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=22016); ap.add_argument("--k", type=int, default=4096)
ap.add_argument("--m", type=int, default=16); ap.add_argument("--split", type=int, default=0)
ap.add_argument("--out", default="f16", choices=["f16", "f32"])
a = ap.parse_args()
W = (torch.randn(a.n, a.k, device="cuda") * 0.02).half()
w = L.Fp6Weight.quantize(W)
x = torch.randn(a.m, a.k, device="cuda").half()
y = torch.empty(a.m, a.n, device="cuda", dtype=torch.float16 if a.out == "f16" else torch.float32)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(4):
    flush.zero_()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); L.w6a16_linear(x, w, out=y, split_k=a.split); e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
lib = _lib.load()
BASE = 0
buf = (ctypes.c_longlong * (256 * 32 + 12 * 64 + 16 * 3 * 64))()
lib.lpqt_trace_dump(buf)
t = np.frombuffer(buf, dtype=np.int64)
plan = L.plan(a.m, a.n, a.k, a.split)
print("shape", a.n, a.k, a.m, "out", a.out, os.environ.get("LPQT_LIB", ""), "plan", plan, "event us (eager, last 3):", [round(v, 2) for v in ts[1:]])
cta = t[BASE:BASE + 256 * 32].reshape(256, 32)[: plan["grid"]].astype(np.float64)
t0 = cta[:, 0].min()
cols = [0, 1, 12, 13, 14, 2, 3, 4, 8, 9, 10, 16, 17, 18, 19, 11, 5, 6]
names = ["entry", "setup", "dq_1st_data", "x_pdl_ok", "mma_1st_x", "prodW_done", "dq0_done", "mma_done",
         "epi_last_dfull", "epi_part_st", "epi_atomic", "fix_divs", "fix_1st_ld", "fix_summed", "fix_stored",
         "epi_fixup", "epi_done", "exit"]
rel = np.where(cta[:, cols] > 0, (cta[:, cols] - t0) / 1e3, np.nan)   # us
for i, n in enumerate(names):
    col = rel[:, i]
    if np.isnan(col).all():
        print(f"{n:>14}: -")
        continue
    print(f"{n:>14}: min {np.nanmin(col):8.2f}  med {np.nanmedian(col):8.2f}  max {np.nanmax(col):8.2f} us"
          f"  (n={int((~np.isnan(col)).sum())})")
print("span entry->last exit: %.2f us" % (np.nanmax(rel[:, -1])))
order = np.argsort(rel[:, -1])[-6:]
print("slowest CTAs: cta smid | " + " ".join(f"{n[:9]:>9}" for n in names))
for c in order:
    print(f"{c:4d} {int(cta[c, 7]):4d} | " + " ".join(f"{v:9.2f}" for v in rel[c]))

ev = t[256 * 32:256 * 32 + 12 * 64].reshape(12, 64)
enames = ["W_issue", "dq_top", "dq_aempty", "dq_sttm", "dq_pre", "dq_waitst", "dq_had_nx", "mma_x_ok", "mma_a_ok",
          "mma_commit"]
base = ev[ev > 0].min() if (ev > 0).any() else 0
print("CTA 0 per-stage clock64 (cycles from first event)")
print("st " + " ".join(f"{n[:10]:>10}" for n in enames))
for i in range(min(40, 64)):
    row = [(ev[e, i] - base) if ev[e, i] > 0 else -1 for e in range(10)]
    print(f"{i:2d} " + " ".join(f"{v:10d}" for v in row))

wt = t[256 * 32 + 12 * 64:].reshape(16, 3, 64)
print("DQ warps, stages 20..27: (aempty_ok, sttm_issued, afull_arrived) relative to warp 0 aempty_ok of the stage")
for i in range(20, 28):
    b = wt[0, 0, i]
    print(f"stage {i}: " + " | ".join(f"w{w}:{wt[w,0,i]-b},{wt[w,1,i]-b},{wt[w,2,i]-b}" for w in range(16)))

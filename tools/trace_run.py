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
ap.add_argument("--events", action="store_true")
a = ap.parse_args()
W = (torch.randn(a.n, a.k, device="cuda") * 0.02).half()
w = L.Fp6Weight.quantize(W)
x = torch.randn(a.m, a.k, device="cuda").half()
y = torch.empty(a.m, a.n, device="cuda", dtype=torch.float16)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(4):
    flush.zero_()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); L.w6a16_linear(x, w, out=y, split_k=a.split); e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
lib = _lib.load()
BASE = 2 * 16 * 64
buf = (ctypes.c_longlong * (BASE + 256 * 8))()
lib.lpqt_trace_dump(buf)
t = np.frombuffer(buf, dtype=np.int64)
plan = L.plan(a.m, a.n, a.k, a.split)
print("shape", a.n, a.k, a.m, "plan", plan, "event us (eager, last 3):", [round(v, 2) for v in ts[1:]])
cta = t[BASE:].reshape(256, 8)[: plan["grid"]].astype(np.float64)
t0 = cta[:, 0].min()
rel = (cta[:, :7] - t0) / 1e3   # us
names = ["entry", "setup", "prodW_done", "dq0_done", "mma_done", "epi_done", "exit"]
for i, n in enumerate(names):
    col = rel[:, i]
    print(f"{n:>11}: min {col.min():8.2f}  med {np.median(col):8.2f}  max {col.max():8.2f} us")
print("span entry->last exit: %.2f us" % (rel[:, 6].max()))
order = np.argsort(rel[:, 6])[-5:]
print("slowest CTAs (cta, smid, entry, setup, prodW, dq, mma, epi, exit):")
for c in order:
    print(c, int(cta[c, 7]), " ".join(f"{v:7.2f}" for v in rel[c]))
if a.events:
    tt = t[:BASE].reshape(2, 16, 64)
    enames = ["p_pre_empty", "p_issued", "dq_it_start", "dq_aempty", "dq_sttm", "dq_pf_full", "dq_waitst",
              "dq_arrive", "mma_ready", "epi_dfull", "mma_commit"]
    for c in range(2):
        base = tt[c][tt[c] > 0].min() if (tt[c] > 0).any() else 0
        print(f"--- CTA {'0' if c == 0 else '77'} (cycles from first event)")
        print("it " + " ".join(f"{n[:11]:>11}" for n in enames))
        for i in range(24):
            row = [(tt[c, e, i] - base) if tt[c, e, i] > 0 else -1 for e in range(11)]
            print(f"{i:2d} " + " ".join(f"{v:11d}" for v in row))
